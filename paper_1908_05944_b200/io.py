"""Canonical serialisation of an ``AlphaComplex`` -- the first "next" row of SURVEY.md 8(f).

``write_complex`` produces exactly the bytes of the reference's ``write_complex``
(reference io.py:228-236) but formats the ~10^7..10^8 lines in C++ host threads
(``axb_format_complex``) instead of a Python loop; ``read_complex`` / ``stats_csv``
mirror reference io.py:239-290.  ``parse_xyzr_arrays`` is the array-native twin of the
reference's ``parse_xyzr`` (io.py:82-101): the same records, comments and
errors, but straight into the ``(n,3)`` / ``(n,)`` float64 arrays the device path uploads -- no
``Ball`` objects (5.6 s per million atoms).  PDB parsing stays out of scope.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

import math

from . import __version__, _native as N
from .errors import AlphaxError, MalformedLine, NonFiniteValue, NonPositiveRadius
from .pipeline import AlphaComplex, complex_stats
from .types import Ball


def _xyzr_slow_scan(text: str):
    """Line-by-line pass with the reference's checks in the reference's order (io.py:85-100);
    only reached when the vectorised pass saw something irregular, to raise the right error."""
    rows = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split()
        if len(parts) != 4:
            raise MalformedLine(lineno, f"expected 4 fields, got {len(parts)}")
        try:
            x, y, z, r = (float(p) for p in parts)
        except ValueError:
            raise MalformedLine(lineno, f"non-numeric field in {raw!r}") from None
        if not all(math.isfinite(v) for v in (x, y, z, r)):
            raise NonFiniteValue(lineno, f"non-finite value in {raw!r}")
        if r <= 0.0:
            raise NonPositiveRadius(lineno, r)
        rows.append((x, y, z, r))
    return np.asarray(rows, dtype=np.float64).reshape(-1, 4)


def parse_xyzr_arrays(text: str):
    """"x y z r" records, one per line, '#' starts a comment (reference io.py:82-101) ->
    ``(centers (n,3) float64, radii (n,) float64)``.  Same values bit for bit (every field goes
    through Python's ``float``), same exceptions with the same line numbers."""
    body = text
    if "#" in body:
        body = "\n".join(raw.split("#", 1)[0] for raw in body.splitlines())
    tokens = body.split()
    table = None
    # fast path: every non-empty line has exactly four tokens <=> token count matches 4 x record lines
    n_lines = sum(1 for raw in body.splitlines() if raw.strip())
    if len(tokens) == 4 * n_lines:
        try:
            table = np.array(tokens, dtype=np.float64).reshape(-1, 4)      # numpy parses like float(): correctly rounded
        except ValueError:
            table = None
        if table is not None and table.size and (not np.isfinite(table).all() or (table[:, 3] <= 0.0).any()):
            table = None
        if table is not None and any(len(raw.split()) not in (0, 4) for raw in body.splitlines()):
            table = None                                                   # e.g. 3 + 5 tokens on two lines
    if table is None:
        table = _xyzr_slow_scan(text)
    return np.ascontiguousarray(table[:, :3]), np.ascontiguousarray(table[:, 3])


def parse_xyzr(text: str) -> list:
    """Reference signature (io.py:82): a list of ``Ball``.  Prefer ``parse_xyzr_arrays`` +
    ``compute_alpha_complex_arrays`` for large inputs."""
    centers, radii = parse_xyzr_arrays(text)
    return [Ball(center=(float(c[0]), float(c[1]), float(c[2])), radius=float(r), index=i)
            for i, (c, r) in enumerate(zip(centers, radii))]


def format_xyzr_arrays(centers, radii) -> str:
    """Inverse of ``parse_xyzr_arrays`` (reference io.py:104-106: ``repr`` of every float)."""
    lines = [f"{float(c[0])!r} {float(c[1])!r} {float(c[2])!r} {float(r)!r}" for c, r in zip(centers, radii)]
    return "\n".join(lines) + ("\n" if lines else "")


def format_xyzr(balls) -> str:
    lines = [f"{b.center[0]!r} {b.center[1]!r} {b.center[2]!r} {b.radius!r}" for b in balls]
    return "\n".join(lines) + ("\n" if lines else "")


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
