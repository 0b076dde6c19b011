"""ctypes binding of libalphax_b200.so -- the C-ABI in include/alphax_b200.h.

There is NO fallback: if the library is missing or CUDA is unavailable the
calls raise ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import NativeLibraryMissing

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libalphax_b200.so")

(OK, ERR_BAD_ARG, ERR_CUDA, ERR_ARENA, ERR_EMPTY, ERR_NONFINITE, ERR_DUPLICATE, ERR_DEGENERATE,
 ERR_BAD_SIDE, ERR_GRID_TOO_LARGE, ERR_DENSITY, ERR_STATE, ERR_INTERNAL) = range(13)

K0, K1, K2, K3, PE, PT, PQ = range(7)
STAGE_KEYS = ("grid", "potential_edges", "potential_triangles", "potential_tets", "prune_tets",
              "prune_triangles", "prune_edges", "prune_vertices", "canonical", "export")

# every symbol include/alphax_b200.h declares
SYMBOLS = (
    "axb_version", "axb_status_name", "axb_ctx_create", "axb_ctx_destroy", "axb_ctx_set_stream",
    "axb_ctx_set_arena", "axb_arena_needed", "axb_arena_used", "axb_arena_hint", "axb_last_message",
    "axb_last_error", "axb_last_error_detail", "axb_grid_build", "axb_grid_build_slab", "axb_slab_rank_range", "axb_merge_rows", "axb_merge_rows_range", "axb_compute_slab",
    "axb_grid_get_info", "axb_grid_export", "axb_potential",
    "axb_potential_counts", "axb_potential_export", "axb_potential_edges", "axb_potential_simplices",
    "axb_potential_import_edges", "axb_potential_import_simplices", "axb_potential_tets_from_triangles", "axb_ac2_mask",
    "axb_sweep_prepare", "axb_sweep_prune", "axb_sweep_rank", "axb_sweep_select",
    "axb_prune", "axb_canonicalize", "axb_export",
    "axb_sync_check", "axb_compute", "axb_compute_into", "axb_compute_start", "axb_compute_finish_into", "axb_compute_host", "axb_export_host", "axb_compute_host_begin",
    "axb_compute_host_finish", "axb_last_d2h_bytes", "axb_stage_ms", "axb_set_stage_timing",
    "axb_kernel_launches", "axb_ortho_batch", "axb_format_complex",
)


class Params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("eps_abs", C.c_double), ("eps_singular", C.c_double),
                ("biomolecule", C.c_int32), ("reserved", C.c_int32)]


class Slab(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("cell_side", C.c_double), ("dims", C.c_int64 * 3),
                ("z_lo", C.c_int64), ("z_hi", C.c_int64)]


class GridInfo(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("cell_side", C.c_double), ("dims", C.c_int64 * 3),
                ("n_cells", C.c_int64), ("n_balls", C.c_int64)]


_lib = None


def load() -> C.CDLL:
    """dlopen the library and declare the prototypes (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is not built (run `python -m paper_1908_05944_b200.build`); "
            "this package has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i64, sz = C.c_void_p, C.c_int64, C.c_size_t
    pi64 = C.POINTER(C.c_int64)
    proto = {
        "axb_version": (C.c_int, []),
        "axb_status_name": (C.c_char_p, [C.c_int]),
        "axb_ctx_create": (C.c_int, [C.POINTER(vp), C.c_int]),
        "axb_ctx_destroy": (None, [vp]),
        "axb_ctx_set_stream": (C.c_int, [vp, vp]),
        "axb_ctx_set_arena": (C.c_int, [vp, vp, sz]),
        "axb_arena_needed": (sz, [vp]),
        "axb_arena_used": (sz, [vp]),
        "axb_arena_hint": (sz, [i64, C.c_double, C.c_double]),
        "axb_last_message": (C.c_char_p, [vp]),
        "axb_last_error": (C.c_int, [vp, C.POINTER(C.c_int), pi64, C.POINTER(C.c_int)]),
        "axb_last_error_detail": (C.c_int, [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
        "axb_grid_build": (C.c_int, [vp, i64, vp, vp, C.POINTER(Params)]),
        "axb_grid_build_slab": (C.c_int, [vp, i64, vp, vp, vp, C.POINTER(Params), C.POINTER(Slab)]),
        "axb_slab_rank_range": (C.c_int, [vp, i64, i64, pi64, pi64]),
        "axb_compute_slab": (C.c_int, [vp, i64, vp, vp, vp, C.POINTER(Params), C.POINTER(Slab), i64, i64, pi64]),
        "axb_merge_rows": (C.c_int, [vp, C.c_int, i64, vp, i64, vp, pi64]),
        "axb_merge_rows_range": (C.c_int, [vp, C.c_int, i64, i64, vp, i64, vp, pi64]),
        "axb_grid_get_info": (C.c_int, [vp, C.POINTER(GridInfo)]),
        "axb_grid_export": (C.c_int, [vp, vp, vp, vp]),
        "axb_potential": (C.c_int, [vp, i64, i64]),
        "axb_potential_counts": (C.c_int, [vp, pi64]),
        "axb_potential_export": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "axb_potential_edges": (C.c_int, [vp, i64, i64]),
        "axb_potential_simplices": (C.c_int, [vp]),
        "axb_potential_import_edges": (C.c_int, [vp, vp, i64]),
        "axb_potential_import_simplices": (C.c_int, [vp, vp, i64, vp, i64]),
        "axb_potential_tets_from_triangles": (C.c_int, [vp, vp, i64]),
        "axb_ac2_mask": (C.c_int, [vp, C.c_int, vp]),
        "axb_sweep_prepare": (C.c_int, [vp]),
        "axb_sweep_prune": (C.c_int, [vp, C.c_double]),
        "axb_sweep_rank": (C.c_int, [vp, C.POINTER(C.c_double), C.c_int]),
        "axb_sweep_select": (C.c_int, [vp, C.c_int]),
        "axb_prune": (C.c_int, [vp]),
        "axb_canonicalize": (C.c_int, [vp, pi64]),
        "axb_export": (C.c_int, [vp, vp, vp, vp, vp]),
        "axb_sync_check": (C.c_int, [vp]),
        "axb_compute": (C.c_int, [vp, i64, vp, vp, C.POINTER(Params), pi64]),
        "axb_compute_into": (C.c_int, [vp, i64, vp, vp, C.POINTER(Params), vp, vp, vp, vp, pi64, pi64]),
        "axb_compute_start": (C.c_int, [vp, i64, vp, vp, C.POINTER(Params)]),
        "axb_compute_finish_into": (C.c_int, [vp, vp, vp, vp, vp, pi64, pi64]),
        "axb_compute_host": (C.c_int, [vp, i64, vp, vp, C.POINTER(Params), pi64]),
        "axb_export_host": (C.c_int, [vp, vp, vp, vp, vp]),
        "axb_compute_host_begin": (C.c_int, [vp, i64, vp, vp, C.POINTER(Params), pi64]),
        "axb_compute_host_finish": (C.c_int, [vp, vp, vp, vp, vp, pi64]),
        "axb_last_d2h_bytes": (i64, [vp]),
        "axb_stage_ms": (C.c_int, [vp, C.POINTER(C.c_float)]),
        "axb_set_stage_timing": (C.c_int, [vp, C.c_int]),
        "axb_kernel_launches": (i64, [vp]),
        "axb_format_complex": (C.c_int, [pi64, vp, vp, vp, vp, vp, i64, pi64]),
        "axb_ortho_batch": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_double, vp, vp, vp]),
    }
    for name, (res, args) in proto.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
