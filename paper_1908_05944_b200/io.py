"""Canonical serialisation of an ``AlphaComplex`` -- the first "next" row of SURVEY.md 8(f).

``write_complex`` produces exactly the bytes of the reference's ``write_complex``
(reference io.py:228-236) but formats the ~10^7..10^8 lines in C++ host threads
(``axb_format_complex``) instead of a Python loop; ``read_complex`` / ``stats_csv``
mirror reference io.py:239-290.  Text parsing of XYZR / PDB inputs stays out of scope.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import __version__, _native as N
from .errors import AlphaxError, MalformedLine
from .pipeline import AlphaComplex, complex_stats


def write_complex(k: AlphaComplex, version: str = __version__) -> str:
    """Header line ``alphax <version> n=<n> alpha=<repr(float)>`` then one line per simplex."""
    lib = N.load()
    arrays = [np.ascontiguousarray(a, dtype=np.int64) for a in (k.vertices, k.edges, k.triangles, k.tets)]
    counts = (C.c_int64 * 4)(*[int(a.shape[0]) for a in arrays])
    ptrs = [a.ctypes.data if a.size else None for a in arrays]
    need = C.c_int64()
    st = lib.axb_format_complex(counts, *ptrs, None, 0, C.byref(need))
    if st != N.OK:
        raise AlphaxError(f"axb_format_complex failed: {lib.axb_status_name(st).decode()}")
    buf = C.create_string_buffer(max(int(need.value), 1))
    st = lib.axb_format_complex(counts, *ptrs, buf, need.value, C.byref(need))
    if st != N.OK:
        raise AlphaxError(f"axb_format_complex failed: {lib.axb_status_name(st).decode()}")
    header = f"alphax {version} n={k.ball_count} alpha={float(k.alpha)!r}\n"
    return header + buf.raw[: need.value].decode("ascii")


def read_complex(text: str) -> AlphaComplex:
    """Inverse of ``write_complex``; validates header, arity, index range and row order."""
    lines = text.splitlines()
    if not lines:
        raise MalformedLine(1, "empty document")
    head = lines[0].split()
    ok = len(head) == 4 and head[0] == "alphax" and head[2].startswith("n=") and head[3].startswith("alpha=")
    try:
        n = int(head[2][2:]) if ok else 0
        alpha = float(head[3][6:]) if ok else 0.0
    except ValueError:
        ok = False
    if not ok:
        raise MalformedLine(1, f"bad header {lines[0]!r}")
    levels = ([], [], [], [])
    for lineno, raw in enumerate(lines[1:], start=2):
        if not raw.strip():
            continue
        try:
            fields = [int(f) for f in raw.split()]
        except ValueError:
            raise MalformedLine(lineno, f"non-integer field in {raw!r}") from None
        dim, verts = fields[0], fields[1:]
        if not 0 <= dim <= 3 or len(verts) != dim + 1:
            raise MalformedLine(lineno, f"bad simplex record {raw!r}")
        if min(verts) < 0 or max(verts) >= n:
            raise MalformedLine(lineno, "vertex index out of range")
        if any(a >= b for a, b in zip(verts, verts[1:])):
            raise MalformedLine(lineno, "vertices must be strictly increasing")
        levels[dim].append(verts)
    return AlphaComplex.from_rows(
        vertices=np.asarray([v[0] for v in levels[0]], dtype=np.int64),
        edges=np.asarray(levels[1], dtype=np.int64).reshape(-1, 2),
        triangles=np.asarray(levels[2], dtype=np.int64).reshape(-1, 3),
        tets=np.asarray(levels[3], dtype=np.int64).reshape(-1, 4),
        alpha=alpha, ball_count=n)


def stats_csv(k: AlphaComplex) -> str:
    """``dim,count`` rows plus ``total`` and ``euler`` (reference io.py:283-290)."""
    st = complex_stats(k)
    rows = ["dim,count"] + [f"{d},{c}" for d, c in enumerate(st.counts)] + [f"total,{st.total}", f"euler,{st.euler}"]
    return "\n".join(rows) + "\n"
