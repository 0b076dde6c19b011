"""Shared helpers for the parity tests."""
import hashlib

import numpy as np


def digest_arrays(*arrays) -> str:
    """sha256 over the int64 bytes of the four simplex arrays (tools/make_golden.py:digest)."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def digest_values(centers, sizes) -> str:
    return hashlib.sha256(np.ascontiguousarray(centers).tobytes() + np.ascontiguousarray(sizes).tobytes()).hexdigest()


def canonical_text(vertices, edges, triangles, tets, n, alpha, version="0.1.0") -> str:
    """The reference's canonical document (reference io.py:228-236), restated for tests."""
    lines = [f"alphax {version} n={n} alpha={float(alpha)!r}"]
    for dim, rows in enumerate((np.asarray(vertices).reshape(-1, 1), edges, triangles, tets)):
        for row in rows:
            lines.append(f"{dim} " + " ".join(str(int(v)) for v in row))
    return "\n".join(lines) + "\n"


def rows_generated_in(levels, rank_of_ball, lo, hi):
    """The rows of a complex (vertices, edges, triangles, tets) whose generator -- the vertex of minimum
    grid rank, reference pipeline.py:10-15 -- has its rank in [lo, hi): what the slab that owns those
    ranks must emit (the slabs of a sharded run partition the complex this way)."""
    out = []
    for d, rows in enumerate(levels):
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, d + 1)
        gen = rank_of_ball[rows].min(axis=1) if rows.shape[0] else np.empty(0, dtype=np.int64)
        sel = rows[(gen >= lo) & (gen < hi)]
        out.append(sel.reshape(-1) if d == 0 else sel)
    return out
