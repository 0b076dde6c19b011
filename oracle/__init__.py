"""CPU oracle for the alpha-complex hot path -- TEST INFRASTRUCTURE ONLY.

ctypes binding of ``libalpha_oracle.so`` (plain-C restatement of the reference
package, see ``alpha_oracle.h``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module; the product package never does.

Parity status: pinned -- ``tests/test_oracle_golden.py`` checks it bit-for-bit
against outputs of the real Python reference (``tests/golden``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libalpha_oracle.so")
_lib = None

OK, EMPTY, NONFINITE, DUPLICATE, DEGENERATE, BAD_SIDE, NOMEM = range(7)
STAGES = ("grid", "potential_edges", "potential_triangles", "potential_tets",
          "prune_tets", "prune_triangles", "prune_edges", "prune_vertices")


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, a second or two)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "alpha_oracle.c"))
    ):
        subprocess.run(["make", "-C", _HERE, "-s", "-B"], check=True)
    return _LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        p64, pd, pu8 = C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_uint8)
        L.axo_ortho_batch.argtypes = [C.c_int64, C.c_int, pd, pd, C.c_double, pd, pd, pu8]
        L.axo_ortho_batch.restype = None
        L.axo_grid_build.argtypes = [C.c_int64, pd, pd, C.c_double, pd, pd, p64, p64, p64, p64]
        L.axo_grid_build.restype = C.c_int
        L.axo_compute.argtypes = [C.c_int64, pd, pd, C.c_double, C.c_double, C.c_double,
                                  C.c_int, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.axo_compute.restype = C.c_int
        L.axo_compute_range.argtypes = [C.c_int64, pd, pd, C.c_double, C.c_double, C.c_double,
                                        C.c_int, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]
        L.axo_compute_range.restype = C.c_int
        L.axo_status.argtypes = [C.c_void_p]
        L.axo_status.restype = C.c_int
        L.axo_error.argtypes = [C.c_void_p, p64, C.POINTER(C.c_int)]
        L.axo_error.restype = None
        L.axo_count.argtypes = [C.c_void_p, C.c_int]
        L.axo_count.restype = C.c_int64
        L.axo_rows.argtypes = [C.c_void_p, C.c_int]
        L.axo_rows.restype = p64
        L.axo_centers.argtypes = [C.c_void_p, C.c_int]
        L.axo_centers.restype = pd
        L.axo_sizes.argtypes = [C.c_void_p, C.c_int]
        L.axo_sizes.restype = pd
        L.axo_stage_seconds.argtypes = [C.c_void_p, pd]
        L.axo_stage_seconds.restype = None
        L.axo_free.argtypes = [C.c_void_p]
        L.axo_free.restype = None
        _lib = L
    return _lib


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _p64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def ortho_batch(points: np.ndarray, r2: np.ndarray, eps_singular: float = 1e-12):
    """(m,k,3), (m,k) -> centres (m,3), sizes (m,), singular (m,) bool."""
    points = np.ascontiguousarray(points, dtype=np.float64)
    r2 = np.ascontiguousarray(r2, dtype=np.float64)
    m, k, _ = points.shape
    cen = np.empty((m, 3), dtype=np.float64)
    siz = np.empty(m, dtype=np.float64)
    sg = np.zeros(m, dtype=np.uint8)
    lib().axo_ortho_batch(m, k, _pd(points), _pd(r2), eps_singular, _pd(cen), _pd(siz),
                          sg.ctypes.data_as(C.POINTER(C.c_uint8)))
    return cen, siz, sg.astype(bool)


@dataclass
class OracleGrid:
    side: float
    origin: np.ndarray
    dims: tuple
    order: np.ndarray
    rank: np.ndarray
    cells: np.ndarray


def grid_build(centers: np.ndarray, radii: np.ndarray, alpha: float):
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    n = centers.shape[0]
    side = C.c_double()
    origin = np.empty(3, dtype=np.float64)
    dims = np.empty(3, dtype=np.int64)
    order = np.empty(n, dtype=np.int64)
    rank = np.empty(n, dtype=np.int64)
    cells = np.empty(n, dtype=np.int64)
    st = lib().axo_grid_build(n, _pd(centers), _pd(radii), float(alpha), C.byref(side), _pd(origin),
                              _p64(dims), _p64(order), _p64(rank), _p64(cells))
    if st != OK:
        return st, None
    return OK, OracleGrid(side.value, origin, tuple(int(d) for d in dims), order, rank, cells)


@dataclass
class OracleResult:
    status: int
    error_vertices: tuple = ()
    vertices: np.ndarray | None = None
    edges: np.ndarray | None = None
    triangles: np.ndarray | None = None
    tets: np.ndarray | None = None
    potentials: dict = field(default_factory=dict)   # dim -> (rows, centres, sizes)
    stage_seconds: dict = field(default_factory=dict)

    def counts(self):
        return (len(self.vertices), len(self.edges), len(self.triangles), len(self.tets))


def compute(centers: np.ndarray, radii: np.ndarray, alpha: float, *, eps_abs: float = 1e-9,
            eps_singular: float = 1e-12, biomolecule: bool = False, chunk: int | None = None,
            threads: int = 1, keep_potentials: bool = False, rank_range: tuple | None = None) -> OracleResult:
    """The whole hot path on the CPU (reference pipeline.py:571-628, mode="grid").
    ``rank_range=(lo, hi)`` computes a single ``_chunk_pass`` over those grid ranks instead."""
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    n = centers.shape[0]
    L = lib()
    h = C.c_void_p()
    if rank_range is not None:
        st = L.axo_compute_range(n, _pd(centers), _pd(radii), float(alpha), float(eps_abs), float(eps_singular),
                                 int(bool(biomolecule)), int(rank_range[0]), int(rank_range[1]), C.byref(h))
    else:
        st = L.axo_compute(n, _pd(centers), _pd(radii), float(alpha), float(eps_abs), float(eps_singular),
                           int(bool(biomolecule)), int(chunk or 0), int(threads), int(bool(keep_potentials)),
                           C.byref(h))
    try:
        verts = (C.c_int64 * 4)()
        nv = C.c_int()
        L.axo_error(h, verts, C.byref(nv))
        out = OracleResult(status=st, error_vertices=tuple(int(verts[i]) for i in range(nv.value)))
        secs = (C.c_double * 8)()
        L.axo_stage_seconds(h, secs)
        out.stage_seconds = {name: float(secs[i]) for i, name in enumerate(STAGES)}
        if st != OK:
            return out

        def rows(what, k):
            m = L.axo_count(h, what)
            if m == 0:
                return np.empty((0, k), dtype=np.int64)
            return np.ctypeslib.as_array(L.axo_rows(h, what), shape=(m, k)).copy()

        out.vertices = rows(0, 1).reshape(-1)
        out.edges = rows(1, 2)
        out.triangles = rows(2, 3)
        out.tets = rows(3, 4)
        if keep_potentials:
            for d in (1, 2, 3):
                what = 3 + d
                m = L.axo_count(h, what)
                if m == 0:
                    out.potentials[d] = (np.empty((0, d + 1), dtype=np.int64), np.empty((0, 3)), np.empty(0))
                else:
                    out.potentials[d] = (
                        rows(what, d + 1),
                        np.ctypeslib.as_array(L.axo_centers(h, what), shape=(m, 3)).copy(),
                        np.ctypeslib.as_array(L.axo_sizes(h, what), shape=(m,)).copy(),
                    )
        return out
    finally:
        L.axo_free(h)
