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

import re

from . import __version__, _native as N
from .errors import AlphaxError, MalformedLine, NonFiniteValue, NonPositiveRadius
from .pipeline import AlphaComplex, complex_stats
from .types import Ball


def _xyzr_record(lineno: int, raw: str):
    """One record line -> (x, y, z, r) or None for a blank / comment line; raises what the reference raises
    for that line (io.py:85-100: field count, then numeric, then finite, then positive radius)."""
    body = raw.partition("#")[0].split()
    if not body:
        return None
    if len(body) != 4:
        raise MalformedLine(lineno, f"expected 4 fields, got {len(body)}")
    try:
        rec = tuple(map(float, body))
    except ValueError:
        raise MalformedLine(lineno, f"non-numeric field in {raw!r}") from None
    if not np.isfinite(rec).all():
        raise NonFiniteValue(lineno, f"non-finite value in {raw!r}")
    if rec[3] <= 0.0:
        raise NonPositiveRadius(lineno, rec[3])
    return rec


def _xyzr_slow_scan(text: str):
    """Record-by-record pass, only reached when the vectorised pass saw something irregular: it exists to
    raise the reference's error for the FIRST offending line (same type, message and line number)."""
    recs = (_xyzr_record(no, raw) for no, raw in enumerate(text.splitlines(), 1))
    return np.array([r for r in recs if r is not None], dtype=np.float64).reshape(-1, 4)


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
    """Reference signature (io.py:104-106) over the array formatter."""
    return format_xyzr_arrays([b.center for b in balls], [b.radius for b in balls])


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


_HEADER = re.compile(r"\s*alphax\s+\S+\s+n=(\S*)\s+alpha=(\S*)\s*\Z")


def _complex_line_error(lineno: int, raw: str, n: int):
    """The reference's verdict on one simplex line (io.py:258-271), in its order of checks."""
    try:
        dim, *verts = (int(f) for f in raw.split())
    except ValueError:
        return MalformedLine(lineno, f"non-integer field in {raw!r}")
    if dim not in (0, 1, 2, 3) or len(verts) != dim + 1:
        return MalformedLine(lineno, f"bad simplex record {raw!r}")
    if not all(0 <= v < n for v in verts):
        return MalformedLine(lineno, "vertex index out of range")
    if sorted(set(verts)) != verts:
        return MalformedLine(lineno, "vertices must be strictly increasing")
    return None


def read_complex(text: str) -> AlphaComplex:
    """Inverse of ``write_complex`` (reference io.py:239-280): validates header, arity, index range and
    strictly increasing rows.  The body is parsed in bulk -- one numpy conversion of all tokens, the checks
    as array operations per dimension -- because a 10^7-simplex document is 10^8 tokens; only when a check
    fails are the lines re-read one by one to raise the reference's error for the first offender."""
    lines = text.splitlines()
    if not lines:
        raise MalformedLine(1, "empty document")
    head = _HEADER.match(lines[0])
    try:
        n, alpha = int(head.group(1)), float(head.group(2))
    except (AttributeError, ValueError):
        raise MalformedLine(1, f"bad header {lines[0]!r}") from None
    body = [(no, raw) for no, raw in enumerate(lines[1:], 2) if raw.strip()]
    levels = None
    try:
        width = np.fromiter((raw.count(" ") + 1 for _, raw in body), dtype=np.int64, count=len(body))
        flat = np.array(" ".join(raw for _, raw in body).split(), dtype=np.int64)
        if flat.size == int(width.sum()):                 # single-space separated records, as write_complex emits them
            start = np.cumsum(width) - width
            dims = flat[start] if len(body) else np.empty(0, dtype=np.int64)
            if ((dims >= 0) & (dims <= 3) & (width == dims + 2)).all():
                levels = []
                for d in range(4):
                    rows = flat[(start[dims == d] + 1)[:, None] + np.arange(d + 1)[None, :]]
                    good = (rows >= 0).all() and (rows < n).all() and (np.diff(rows, axis=1) > 0).all()
                    if not good:
                        levels = None
                        break
                    levels.append(rows)
    except (ValueError, OverflowError):
        levels = None
    if levels is None:                                    # irregular spacing or a bad record: line by line
        levels = [[], [], [], []]
        for no, raw in body:
            err = _complex_line_error(no, raw, n)
            if err is not None:
                raise err
            dim, *verts = (int(f) for f in raw.split())
            levels[dim].append(verts)
        levels = [np.asarray(lv, dtype=np.int64).reshape(-1, d + 1) for d, lv in enumerate(levels)]
    return AlphaComplex.from_rows(vertices=levels[0].reshape(-1), edges=levels[1], triangles=levels[2],
                                  tets=levels[3], alpha=alpha, ball_count=n)


def stats_csv(k: AlphaComplex) -> str:
    """``dim,count`` rows plus ``total`` and ``euler`` (reference io.py:283-290)."""
    st = complex_stats(k)
    rows = ["dim,count"] + [f"{d},{c}" for d, c in enumerate(st.counts)] + [f"total,{st.total}", f"euler,{st.euler}"]
    return "\n".join(rows) + "\n"
