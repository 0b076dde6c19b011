"""Host side of the drop-in boundary: ``compute_alpha_complex`` on a B200.

Mirrors the reference's public interface for the hot path (reference
pkg/src/alphax/pipeline.py): ``PipelineConfig`` (:55-83), ``AlphaComplex``
(:117-187), ``complex_stats`` (:197-200), ``closure_ok`` (:203-211),
``compute_alpha_complex(balls, cfg, stage_times=None)`` (:571-628).  All
geometry runs in hand-written CUDA kernels behind the C-ABI of
``include/alphax_b200.h``; this module only validates arguments, moves
buffers (torch owns device memory and streams) and maps status codes back to
the reference's exceptions.  There is no CPU fallback.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Iterator, Sequence

import numpy as np

from . import _native as N
from .errors import (AlphaxError, DegenerateSimplex, DuplicateCenter, EmptyInput, NativeLibraryMissing,
                     NonFiniteCoordinate, UnsupportedMode)
from .types import Ball, SimplexKey, TolerancePolicy

STAGE_NAMES = ("grid", "potential_edges", "potential_triangles", "potential_tets",
               "prune_tets", "prune_triangles", "prune_edges", "io")


@dataclass(frozen=True)
class PipelineConfig:
    """Run configuration (reference pipeline.py:55-83).

    ``alpha`` is in A^2 and compared as ``size <= alpha + eps_abs``.
    ``chunk_size`` and ``workers`` are accepted for drop-in compatibility and
    ignored: the result is provably independent of them (reference
    T/test_acceptance.py:218-233) and the GPU schedules its own work.
    """

    alpha: float
    mode: str = "grid"
    chunk_size: int | None = None
    workers: int = 1
    biomolecule_mode: bool = False
    tolerance: TolerancePolicy = field(default_factory=TolerancePolicy)

    def __post_init__(self):
        if not np.isfinite(self.alpha):
            raise ValueError("alpha must be finite")
        if self.mode not in ("grid", "naive"):
            raise ValueError(f"mode must be 'grid' or 'naive', got {self.mode!r}")
        if self.chunk_size is not None and self.chunk_size < 1:
            raise ValueError("chunk_size must be positive")
        if self.workers < 1:
            raise ValueError("workers must be positive")
        if self.biomolecule_mode and self.alpha < 0.0:
            raise ValueError("biomolecule_mode requires alpha >= 0")


def _rows_view(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a.view([("", np.int64)] * a.shape[1]).ravel()


def _rows_isin(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    if a.shape[0] == 0 or b.shape[0] == 0:
        return np.zeros(a.shape[0], dtype=bool)
    return np.isin(_rows_view(a), _rows_view(b))


def _canonical_rows(a, k: int) -> np.ndarray:
    a = np.asarray(a, dtype=np.int64).reshape(-1, k)
    return np.unique(a, axis=0) if a.shape[0] else a.copy()


@dataclass(frozen=True, eq=False)
class AlphaComplex:
    """The result container of the reference (pipeline.py:117-187): vertices
    (k0,) ascending; edges/triangles/tets (k, d+1) int64 rows, each strictly
    increasing, rows in lexicographic order, no duplicates."""

    vertices: np.ndarray
    edges: np.ndarray
    triangles: np.ndarray
    tets: np.ndarray
    alpha: float
    ball_count: int

    @classmethod
    def from_rows(cls, vertices, edges, triangles, tets, alpha, ball_count) -> "AlphaComplex":
        return cls(vertices=np.unique(np.asarray(vertices, dtype=np.int64)), edges=_canonical_rows(edges, 2),
                   triangles=_canonical_rows(triangles, 3), tets=_canonical_rows(tets, 4),
                   alpha=float(alpha), ball_count=int(ball_count))

    def level(self, dim: int) -> np.ndarray:
        if dim == 0:
            return self.vertices.reshape(-1, 1)
        return (self.edges, self.triangles, self.tets)[dim - 1]

    def counts(self) -> tuple:
        return tuple(int(self.level(d).shape[0]) for d in range(4))

    @property
    def total(self) -> int:
        return sum(self.counts())

    def simplex_keys(self, dim: int) -> list:
        return [SimplexKey(tuple(int(v) for v in row)) for row in self.level(dim)]

    def iter_simplices(self) -> Iterator[SimplexKey]:
        for dim in range(4):
            yield from self.simplex_keys(dim)

    def contains(self, key: SimplexKey) -> bool:
        probe = np.asarray([key.vertices], dtype=np.int64)
        return bool(_rows_isin(probe, self.level(key.dim))[0])

    def __eq__(self, other) -> bool:
        if not isinstance(other, AlphaComplex):
            return NotImplemented
        if self.ball_count != other.ball_count or self.alpha != other.alpha:
            return False
        return all(np.array_equal(self.level(d), other.level(d)) for d in range(4))

    def symmetric_difference(self, other: "AlphaComplex") -> dict:
        """dim -> (rows only in self, rows only in other)."""
        diff = {}
        for d in range(4):
            mine, theirs = self.level(d), other.level(d)
            diff[d] = (mine[~_rows_isin(mine, theirs)], theirs[~_rows_isin(theirs, mine)])
        return diff

    def is_subcomplex_of(self, other: "AlphaComplex") -> bool:
        return all(bool(_rows_isin(self.level(d), other.level(d)).all()) for d in range(4))


@dataclass(frozen=True)
class ComplexStats:
    counts: tuple
    total: int
    euler: int


def complex_stats(k: AlphaComplex) -> ComplexStats:
    c = k.counts()
    return ComplexStats(counts=c, total=sum(c), euler=c[0] - c[1] + c[2] - c[3])


def _facets(rows: np.ndarray) -> np.ndarray:
    k = rows.shape[1]
    return np.concatenate([np.delete(rows, drop, axis=1) for drop in range(k)], axis=0)


def closure_ok(k: AlphaComplex) -> bool:
    """Every facet of every simplex is a member (reference pipeline.py:203-211).
    Host-side numpy check for tests and debugging; the device pipeline
    guarantees closure by construction (kept simplices mark all their faces)."""
    if k.tets.size and not _rows_isin(np.unique(_facets(k.tets), axis=0), k.triangles).all():
        return False
    if k.triangles.size and not _rows_isin(np.unique(_facets(k.triangles), axis=0), k.edges).all():
        return False
    if k.edges.size and not np.isin(np.unique(k.edges), k.vertices).all():
        return False
    return True


# --------------------------------------------------------------------------- engine


class Engine:
    """One CUDA context of the native library on one GPU: owns the scratch
    arena (a torch uint8 tensor) and maps status codes to exceptions."""

    def __init__(self, device: int | None = None, arena_bytes: int = 0):
        import torch

        if not torch.cuda.is_available():
            raise NativeLibraryMissing("CUDA is not available; this package has no CPU fallback")
        self.torch = torch
        self.lib = N.load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._device_str = f"cuda:{self.device}"
        self.handle = C.c_void_p()
        st = self.lib.axb_ctx_create(C.byref(self.handle), self.device)
        if st != N.OK:
            raise AlphaxError(f"axb_ctx_create failed: {self.lib.axb_status_name(st).decode()}")
        self.arena = None
        self._stage_ms: dict = {}
        self._stage_ms_stale = False
        self._stage_timing = False
        # identity of what is resident on the device, for the stage API's handles (stages.py): a new token for every
        # run that rebuilds the grid, a new id for every edge level / simplex level computed or imported
        self._remembered_counts: dict = {}     # (n, configuration) -> row counts of the last result (compute_device)
        self._host_caps: dict = {}           # compute_host: capacities of the last call per problem shape
        self.token = 0
        self.edge_id = 0
        self.simplex_id = 0
        self.stage_key = None
        if arena_bytes:
            self._set_arena(arena_bytes)

    def close(self):
        if self.handle:
            self.lib.axb_ctx_destroy(self.handle)
            self.handle = C.c_void_p()
        self.arena = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    def _set_arena(self, nbytes: int):
        torch = self.torch
        self.arena = None          # free before growing
        nbytes = (int(nbytes) + 4095) // 4096 * 4096
        self.arena = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        st = self.lib.axb_ctx_set_arena(self.handle, self.arena.data_ptr(), nbytes)
        if st != N.OK:
            raise AlphaxError(self._message())

    def _bind_stream(self, fresh: bool = True):
        """fresh: the call rebuilds the device state from the inputs, so handles of the stage API go stale."""
        if fresh:
            self.token += 1
            self.stage_key = None
        stream = self.torch.cuda.current_stream(self.device)
        self.lib.axb_ctx_set_stream(self.handle, C.c_void_p(stream.cuda_stream))

    def _message(self) -> str:
        return self.lib.axb_last_message(self.handle).decode(errors="replace")

    def _params(self, cfg: PipelineConfig) -> N.Params:
        return N.Params(float(cfg.alpha), float(cfg.tolerance.eps_abs), float(cfg.tolerance.eps_singular),
                        1 if cfg.biomolecule_mode else 0, 0)

    def _error_vertices(self):
        verts = (C.c_int64 * 4)()
        nv = C.c_int()
        st = C.c_int()
        self.lib.axb_last_error(self.handle, C.byref(st), verts, C.byref(nv))
        return tuple(int(verts[i]) for i in range(nv.value))

    def _error_detail(self):
        key = C.c_uint64()
        xyz = (C.c_double * 3)()
        self.lib.axb_last_error_detail(self.handle, C.byref(key), xyz)
        return int(key.value), tuple(float(v) for v in xyz)

    def _raise(self, st: int, cfg: PipelineConfig, centers=None, radii=None):
        """Status -> the exception the reference raises for the same input."""
        if st == N.ERR_EMPTY:
            raise EmptyInput("at least one ball is required")
        if st == N.ERR_NONFINITE:
            raise NonFiniteCoordinate(f"ball {self._error_vertices()[0]} is not finite")
        if st == N.ERR_DUPLICATE:
            i, j = self._error_vertices()
            raise DuplicateCenter(f"balls {i} and {j} share the center {self._error_detail()[1]}")
        if st == N.ERR_DEGENERATE:
            bad = self._error_vertices()
            what = {2: "edge", 3: "triangle", 4: "tetrahedron"}.get(len(bad), "simplex")
            raise DegenerateSimplex(f"{what} {bad} has affinely dependent centers", vertices=bad)
        if st == N.ERR_BAD_SIDE:
            r_max = float(_max_to_host(radii)) if radii is not None else float("nan")
            raise ValueError(f"alpha={cfg.alpha} gives non-positive squared cell side (r_max={r_max})")
        name = self.lib.axb_status_name(st).decode()
        raise AlphaxError(f"{name}: {self._message()}")

    def raise_slab_error(self, rec, cfg: PipelineConfig):
        """The exception for a `sharding.SlabError` every rank agreed on (same types and messages as _raise)."""
        st, verts = rec.status, tuple(rec.vertices)
        if st == N.ERR_NONFINITE:
            raise NonFiniteCoordinate(f"ball {verts[0]} is not finite")
        if st == N.ERR_DUPLICATE:
            raise DuplicateCenter(f"balls {verts[0]} and {verts[1]} share the center {tuple(rec.xyz)}")
        if st == N.ERR_DEGENERATE:
            what = {2: "edge", 3: "triangle", 4: "tetrahedron"}.get(len(verts), "simplex")
            raise DegenerateSimplex(f"{what} {verts} has affinely dependent centers", vertices=verts)
        if st == N.ERR_BAD_SIDE:
            raise ValueError(f"alpha={cfg.alpha} gives non-positive squared cell side")
        name = self.lib.axb_status_name(st).decode()
        raise AlphaxError(f"{name}: {rec.message or 'reported by another rank'}")

    def _with_arena(self, n: int, alpha: float, call):
        """Run ``call()`` (returns a status), growing the arena on AXB_ERR_ARENA: the library reports the size that
        would have sufficed, so the second attempt normally fits."""
        if self.arena is None:
            self._set_arena(self.lib.axb_arena_hint(n, float(alpha), 1.9))
        for _ in range(12):
            st = call()
            if st != N.ERR_ARENA:
                return st
            need = int(self.lib.axb_arena_needed(self.handle))
            have = self.arena.numel()
            self._set_arena(max(int(need * 1.3) + (64 << 20), int(have * 1.5)))
        raise AlphaxError("scratch arena kept overflowing: " + self._message())

    def _collect_stage_ms(self):
        # read on demand: ten cudaEventElapsedTime calls cost ~30 us, which the GPU would spend idle between two calls
        self._stage_ms_stale = True

    @property
    def stage_timing(self) -> bool:
        """Whether the runs of this engine bracket their stages with CUDA events (``last_stage_ms``).  Off by default,
        like the reference's ``stage_times=None``: the event records cost 0.04-0.06 ms per run."""
        return self._stage_timing

    @stage_timing.setter
    def stage_timing(self, on: bool):
        self._stage_timing = bool(on)
        self.lib.axb_set_stage_timing(self.handle, int(self._stage_timing))

    @contextlib.contextmanager
    def timing_stages(self, on: bool = True):
        """``with eng.timing_stages(): ...`` -- stage timing for the calls inside, the previous setting afterwards."""
        before = self._stage_timing
        self.stage_timing = on
        try:
            yield self
        finally:
            self.stage_timing = before

    @property
    def last_stage_ms(self) -> dict:
        """Device time per stage of the most recent call (CUDA events; the reference's stage_times keys); zeros
        unless ``stage_timing`` was on for that call."""
        if self._stage_ms_stale:
            ms = (C.c_float * len(N.STAGE_KEYS))()
            self.lib.axb_stage_ms(self.handle, ms)
            self._stage_ms = {k: float(ms[i]) for i, k in enumerate(N.STAGE_KEYS)}
            self._stage_ms_stale = False
        return self._stage_ms

    @last_stage_ms.setter
    def last_stage_ms(self, value: dict):
        self._stage_ms = dict(value)
        self._stage_ms_stale = False

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.axb_kernel_launches(self.handle))

    # -- the hot path
    def compute_host(self, centers: np.ndarray, radii: np.ndarray, cfg: PipelineConfig, pinned_out: bool = True,
                     pipelined: bool = True):
        """Host arrays in, four host int64 arrays out (H2D and D2H inside).

        ``pipelined``: the result arrays are allocated from tight capacity bounds known after the
        potential stage (``axb_compute_host_begin``) and every dimension is copied to the host as soon
        as it is final, overlapping the remaining kernels (``axb_compute_host_finish``); the returned
        arrays are then leading slices of slightly larger pinned buffers.  Otherwise (or if a bound did
        not hold) the plain two-call path ``axb_compute_host`` + ``axb_export_host`` is used."""
        torch = self.torch
        centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
        radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
        n = centers.shape[0]
        if radii.shape[0] != n:
            raise ValueError("centers and radii disagree in length")
        if n == 0:
            raise EmptyInput("at least one ball is required")
        prm = self._params(cfg)
        counts = (C.c_int64 * 4)()
        outs: list = []

        def host_arrays(rows):
            outs.clear()
            for d in range(4):
                shape = (int(rows[d]),) if d == 0 else (int(rows[d]), d + 1)
                if pinned_out and rows[d]:
                    outs.append(torch.empty(shape, dtype=torch.int64, pin_memory=True).numpy())
                else:
                    outs.append(np.empty(shape, dtype=np.int64))

        def run_two_calls():
            st = self.lib.axb_compute_host(self.handle, n, centers.ctypes.data, radii.ctypes.data, C.byref(prm), counts)
            if st != N.OK:
                return st
            host_arrays(counts)
            # an arena overflow here re-runs the whole computation with a larger arena
            return self.lib.axb_export_host(self.handle, *(o.ctypes.data if o.size else None for o in outs))

        shape_key = (n, float(cfg.alpha), float(cfg.tolerance.eps_abs), float(cfg.tolerance.eps_singular), bool(cfg.biomolecule_mode))

        def run_pipelined():
            cap = (C.c_int64 * 4)()
            # the result arrays of a repeated problem shape are allocated BEFORE the GPU is started (2 % above the last
            # capacities), so nothing but the call overhead lies between `begin` and `finish`, where the GPU waits
            prev = self._host_caps.get(shape_key)
            if prev is not None:
                host_arrays(prev)
            st = self.lib.axb_compute_host_begin(self.handle, n, centers.ctypes.data, radii.ctypes.data, C.byref(prm), cap)
            if st != N.OK:
                return st
            # (the first call of a shape allocates the same 2 % above the bounds that the later ones ask for: the pinned
            # caching allocator then hands the same blocks out again -- a fresh 1.8 GB cudaHostAlloc at 10M atoms is 0.9 s)
            want = tuple(min(n, int(cap[d])) if d == 0 else int(cap[d]) + int(cap[d]) // 50 for d in range(4))
            if prev is None or any(int(cap[d]) > prev[d] for d in range(4)):
                host_arrays(want)
            self._host_caps[shape_key] = want
            if len(self._host_caps) > 64:
                self._host_caps.pop(next(iter(self._host_caps)))
            st = self.lib.axb_compute_host_finish(self.handle, *(o.ctypes.data if o.size else None for o in outs), counts)
            if st == N.OK:
                outs[:] = [o[: int(counts[d])] for d, o in enumerate(outs)]
            return st

        with torch.cuda.device(self.device):
            self._bind_stream()
            st = self._with_arena(n, cfg.alpha, run_pipelined if pipelined else run_two_calls)
            if st == N.ERR_STATE and pipelined:
                st = self._with_arena(n, cfg.alpha, run_two_calls)
            if st != N.OK:
                self._raise(st, cfg, centers, radii)
            self._collect_stage_ms()
        return outs

    def compute_device(self, centers, radii, cfg: PipelineConfig):
        """CUDA tensors in (centers (n,3) f64, radii (n,) f64), four CUDA int64 tensors out.

        The first call for a problem shape runs ``axb_compute`` (which ends with the row counts on the host), allocates the
        lists and runs ``axb_export``.  It remembers the counts; the next call with the same (n, configuration) --
        another frame of a trajectory, the next step of a benchmark -- runs ``axb_compute_start``, allocates 2 % above
        them while the GPU works, and ``axb_compute_finish_into``: nothing waits for the host between the pruning stage
        and the last row.  If a list outgrew its buffer the first form is used again."""
        torch = self.torch
        if centers.dtype != torch.float64 or centers.dim() != 2 or not centers.is_contiguous():
            centers = centers.to(dtype=torch.float64).contiguous().reshape(-1, 3)
        if radii.dtype != torch.float64 or radii.dim() != 1 or not radii.is_contiguous():
            radii = radii.to(dtype=torch.float64).contiguous().reshape(-1)
        n = centers.shape[0]
        if n == 0:
            raise EmptyInput("at least one ball is required")
        prm = self._params(cfg)
        counts = (C.c_int64 * 4)()
        dev = self._device_str
        shape_key = (n, float(cfg.alpha), float(cfg.tolerance.eps_abs), float(cfg.tolerance.eps_singular), bool(cfg.biomolecule_mode))

        def carve(flat, rows):
            outs, at = [], 0
            for d in range(4):
                part = flat[at:at + rows[d] * (d + 1)]
                outs.append(part if d == 0 else part.view(rows[d], d + 1))
                at += rows[d] * (d + 1)
            return outs

        with torch.cuda.device(self.device):
            self._bind_stream()
            last = self._remembered_counts.get(shape_key)
            if last is not None:
                cap = [min(n, last[0] + last[0] // 50 + 64)] + [last[d] + last[d] // 50 + 1024 for d in (1, 2, 3)]
                ccap = (C.c_int64 * 4)(*cap)
                bufs = None

                def run_warm():
                    nonlocal bufs
                    st = self.lib.axb_compute_start(self.handle, n, centers.data_ptr(), radii.data_ptr(), C.byref(prm))
                    if st != N.OK:
                        return st
                    if bufs is None:                   # allocated while the triangle / tet and pruning kernels run
                        bufs = carve(torch.empty(sum(cap[d] * (d + 1) for d in range(4)), dtype=torch.int64, device=dev), cap)
                    return self.lib.axb_compute_finish_into(self.handle, *(b.data_ptr() for b in bufs), ccap, counts)

                st = self._with_arena(n, cfg.alpha, run_warm)
                if st == N.OK:
                    self._remembered_counts[shape_key] = tuple(int(v) for v in counts)
                    self._collect_stage_ms()
                    return [b[: int(counts[d])] for d, b in enumerate(bufs)]
                if st != N.ERR_STATE:
                    self._raise(st, cfg, centers, radii)
                del bufs                                   # a list outgrew its buffer: the two-call form below
            st = self._with_arena(n, cfg.alpha, lambda: self.lib.axb_compute(
                self.handle, n, centers.data_ptr(), radii.data_ptr(), C.byref(prm), counts))
            if st != N.OK:
                self._raise(st, cfg, centers, radii)
            # one allocation for the four lists (the GPU idles while the host allocates: every call counts)
            rows = [int(counts[d]) for d in range(4)]
            outs = carve(torch.empty(sum(rows[d] * (d + 1) for d in range(4)), dtype=torch.int64, device=dev), rows)
            st = self.lib.axb_export(self.handle, *(o.data_ptr() if o.numel() else None for o in outs))
            if st == N.OK:
                st = self.lib.axb_sync_check(self.handle)
            if st != N.OK:
                self._raise(st, cfg, centers, radii)
            self._remembered_counts[shape_key] = tuple(rows)
            if len(self._remembered_counts) > 64:
                self._remembered_counts.pop(next(iter(self._remembered_counts)))
            self._collect_stage_ms()
        return outs


    # -- stage-by-stage access (the reference's standalone stage operations, pipeline.py:640-731).
    # The arena must already be large enough: growing it would drop the state of earlier stages.
    def _check(self, st, cfg, centers=None, radii=None):
        if st != N.OK:
            self._raise(st, cfg, centers, radii)

    def stage_grid(self, centers, radii, cfg: PipelineConfig, arena_factor: float = 4.0, key=None):
        """validate_input + build_grid_arrays on CUDA tensors; returns the grid geometry.
        key: what the caller wants to recognise this device state by later (stages.py)."""
        torch = self.torch
        self._stage_inputs = (centers.to(dtype=torch.float64).contiguous().reshape(-1, 3),
                              radii.to(dtype=torch.float64).contiguous().reshape(-1))
        self._stage_cfg = cfg
        n = self._stage_inputs[0].shape[0]
        want = int(self.lib.axb_arena_hint(max(n, 1), float(cfg.alpha), 1.9) * arena_factor)
        if self.arena is None or self.arena.numel() < want:
            self._set_arena(want)
        prm = self._params(cfg)
        with torch.cuda.device(self.device):
            self._bind_stream()
            st = self.lib.axb_grid_build(self.handle, n, self._stage_inputs[0].data_ptr(),
                                         self._stage_inputs[1].data_ptr(), C.byref(prm))
        self._check(st, cfg, *self._stage_inputs)
        self.stage_key = key
        info = N.GridInfo()
        self.lib.axb_grid_get_info(self.handle, C.byref(info))
        return dict(origin=np.array(list(info.origin)), cell_side=float(info.cell_side),
                    dims=tuple(int(d) for d in info.dims), n_cells=int(info.n_cells), n_balls=int(info.n_balls))

    def stage_grid_export(self):
        torch = self.torch
        n = self._stage_inputs[0].shape[0]
        out = [torch.empty(n, dtype=torch.int64, device=f"cuda:{self.device}") for _ in range(3)]
        self._check(self.lib.axb_grid_export(self.handle, *(o.data_ptr() for o in out)), self._stage_cfg)
        return out      # order, rank, ball_cells

    def _stage_call(self, fn, *args):
        with self.torch.cuda.device(self.device):
            self._bind_stream(fresh=False)
            st = fn(self.handle, *args)
        self._check(st, self._stage_cfg, *self._stage_inputs)

    def _rows_arg(self, rows, k: int):
        torch = self.torch
        t = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int64).reshape(-1, k) if isinstance(rows, np.ndarray) else rows,
                            device=f"cuda:{self.device}").to(dtype=torch.int64).contiguous().reshape(-1, k)
        return t, (t.data_ptr() if t.shape[0] else None), int(t.shape[0])

    def stage_potential(self, lo: int = 0, hi: int | None = None):
        """All three potential levels for the generators at grid ranks [lo, hi) (one reference chunk)."""
        n = self._stage_inputs[0].shape[0]
        self._stage_call(self.lib.axb_potential, int(lo), int(n if hi is None else hi))
        self.edge_id += 1
        self.simplex_id += 1
        return self.stage_potential_counts()

    def stage_potential_counts(self):
        counts = (C.c_int64 * 3)()
        self.lib.axb_potential_counts(self.handle, counts)
        return tuple(int(v) for v in counts)

    def stage_edges(self, lo: int = 0, hi: int | None = None):
        """Stage one alone (potential_edges, pipeline.py:640-646); the level stays resident."""
        n = self._stage_inputs[0].shape[0]
        self._stage_call(self.lib.axb_potential_edges, int(lo), int(n if hi is None else hi))
        self.edge_id += 1
        return self.stage_potential_counts()[0]

    def stage_import_edges(self, rows):
        """Replace the resident edge level by caller rows (m, 2) of ball indices."""
        keep, ptr, m = self._rows_arg(rows, 2)
        self._stage_call(self.lib.axb_potential_import_edges, ptr, m)
        self.edge_id += 1

    def stage_simplices(self):
        """Potential triangles + tets from the resident edge level."""
        self._stage_call(self.lib.axb_potential_simplices)
        self.simplex_id += 1
        return self.stage_potential_counts()

    def stage_import_simplices(self, tri_rows, tet_rows):
        kt, pt, mt = self._rows_arg(tri_rows, 3)
        kq, pq, mq = self._rows_arg(tet_rows, 4)
        self._stage_call(self.lib.axb_potential_import_simplices, pt, mt, pq, mq)
        self.simplex_id += 1

    def stage_tets_from_triangles(self, tri_rows):
        """The reference's standalone potential_tets (pipeline.py:670-709) on caller triangle rows."""
        kt, pt, mt = self._rows_arg(tri_rows, 3)
        self._stage_call(self.lib.axb_potential_tets_from_triangles, pt, mt)
        self.simplex_id += 1
        return self.stage_potential_counts()

    def stage_ac2_mask(self, dim: int):
        """_ac2_mask (pipeline.py:286-313) of the resident potential level `dim`, in stage_potential_export's row order."""
        torch = self.torch
        m = self.stage_potential_counts()[dim - 1]
        mask = torch.empty(m, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._stage_call(self.lib.axb_ac2_mask, N.PE + dim - 1, mask.data_ptr() if m else None)
        return mask.to(torch.bool)

    def stage_potential_export(self, dim: int):
        """(rows, centres, sizes) of one potential level as CUDA tensors, in generation order."""
        torch = self.torch
        m = self.stage_potential_counts()[dim - 1]
        dev = f"cuda:{self.device}"
        rows = torch.empty((m, dim + 1), dtype=torch.int64, device=dev)
        cen = torch.empty((m, 3), dtype=torch.float64, device=dev)
        siz = torch.empty(m, dtype=torch.float64, device=dev)
        self._stage_call(self.lib.axb_potential_export, N.PE + dim - 1, rows.data_ptr() if m else None,
                         cen.data_ptr() if m else None, siz.data_ptr() if m else None)
        return rows, cen, siz

    def stage_prune(self):
        self._stage_call(self.lib.axb_prune)

    def stage_canonicalize(self):
        counts = (C.c_int64 * 4)()
        self._stage_call(self.lib.axb_canonicalize, counts)
        return tuple(int(v) for v in counts)

    def stage_export(self, counts):
        torch = self.torch
        dev = f"cuda:{self.device}"
        outs = [torch.empty((int(counts[d]),) if d == 0 else (int(counts[d]), d + 1), dtype=torch.int64, device=dev)
                for d in range(4)]
        self._stage_call(self.lib.axb_export, *(o.data_ptr() if o.numel() else None for o in outs))
        self._stage_call(self.lib.axb_sync_check)
        self._collect_stage_ms()
        return outs

    # -- alpha sweep with re-use (csrc/sweep.cuh)
    def sweep_device(self, centers, radii, alphas, cfg: PipelineConfig):
        """The complexes of ONE ball set at several alphas: grid, potential levels, ortho solves and every AC2 walk
        are done once at max(alphas); each alpha then costs one flag pass over the listed edges, the inheritance marks
        and the canonical lists.  CUDA tensors in, a list (one entry per alpha, in the given order) of four CUDA int64
        tensors out -- bit-identical to independent runs.  ``cfg.alpha`` is ignored."""
        from dataclasses import replace

        alphas = [float(a) for a in alphas]
        if not alphas:
            return []
        top = replace(cfg, alpha=max(alphas))
        self.stage_grid(centers, radii, top)
        self.stage_potential()
        self._stage_call(self.lib.axb_sweep_prepare)
        # the sweep as a filtration: every listed simplex gets the index of the first alpha that keeps it, once; each
        # alpha is then one threshold pass (axb_sweep_select).  Fallback (a face of a listed tet that rounding left
        # unlisted, or more than 254 alphas): the pruning kernels per alpha on the prepared arrays (axb_sweep_prune).
        ranked = sorted(set(alphas))
        use_ranks = len(ranked) <= 254
        if use_ranks:
            arr = (C.c_double * len(ranked))(*ranked)
            with self.torch.cuda.device(self.device):
                self._bind_stream(fresh=False)
                st = self.lib.axb_sweep_rank(self.handle, arr, len(ranked))
            if st == N.ERR_STATE:
                use_ranks = False
            else:
                self._check(st, self._stage_cfg, *self._stage_inputs)
        out = []
        for a in alphas:
            if use_ranks:
                self._stage_call(self.lib.axb_sweep_select, ranked.index(a))
            else:
                self._stage_call(self.lib.axb_sweep_prune, C.c_double(a))
            out.append(self.stage_export(self.stage_canonicalize()))
        return out

    # -- multi-GPU building blocks (sharding.py)
    def compute_slab_device(self, centers, radii, global_index, cfg: PipelineConfig, plan, slab, raise_errors: bool = True):
        """One z-slab of a global grid: CUDA tensors of the loaded balls (ascending global index) in,
        the four row lists in GLOBAL ball indices out -- the kept simplices whose generator lies in an
        owned layer, disjoint from every other slab's.  raise_errors=False returns (rows, SlabError | None)
        instead of raising (error vertices are global ball indices, the key is shifted to global grid ranks)."""
        torch = self.torch
        n = int(radii.shape[0])
        prm = self._params(cfg)
        geo = N.Slab((C.c_double * 3)(*[float(v) for v in plan.origin]), float(plan.cell_side),
                     (C.c_int64 * 3)(*[int(v) for v in plan.dims]), int(slab.z_lo), int(slab.z_hi))
        dev = f"cuda:{self.device}"
        outs: list = []

        def run():
            lib, h = self.lib, self.handle
            counts = (C.c_int64 * 4)()
            st = lib.axb_compute_slab(h, n, centers.data_ptr(), radii.data_ptr(), global_index.data_ptr(), C.byref(prm),
                                      C.byref(geo), int(slab.z_own_lo), int(slab.z_own_hi), counts)
            if st != N.OK:
                return st
            outs.clear()
            outs.extend(torch.empty((int(counts[d]),) if d == 0 else (int(counts[d]), d + 1), dtype=torch.int64,
                                    device=dev) for d in range(4))
            st = lib.axb_export(h, *(o.data_ptr() if o.numel() else None for o in outs))
            return st if st != N.OK else lib.axb_sync_check(h)

        with torch.cuda.device(self.device):
            self._bind_stream()
            st = self._with_arena(n, cfg.alpha, run)
        if st != N.OK:
            if raise_errors:
                self._raise(st, cfg, centers, radii)
            from .sharding import SlabError

            key, xyz = self._error_detail()
            if st == N.ERR_DEGENERATE:
                key += int(slab.first_rank) << 29      # ERR_ORD_BITS of csrc/common.cuh
            return [], SlabError(status=int(st), key=key, vertices=self._error_vertices(), xyz=xyz, message=self._message())
        self._collect_stage_ms()
        return outs if raise_errors else (outs, None)

    def merge_rows(self, rows, k: int, n_index: int, index_lo: int = 0):
        """Sorted duplicate-free union of canonical rows (CUDA int64 tensor (m,k) or (m,) for k=1) whose first index
        lies in [index_lo, n_index)."""
        torch = self.torch
        rows = rows.contiguous().reshape(-1, k)
        m = int(rows.shape[0])
        if m == 0:
            return rows.reshape(-1) if k == 1 else rows
        out = torch.empty((m, k), dtype=torch.int64, device=rows.device)
        count = C.c_int64()

        def run():
            return self.lib.axb_merge_rows_range(self.handle, k, int(index_lo), int(n_index), rows.data_ptr() if m else None, m,
                                                 out.data_ptr() if m else None, C.byref(count))

        with torch.cuda.device(self.device):
            self._bind_stream()
            st = self._with_arena(max(m, n_index - index_lo) // 8 + 1, 0.0, run)
        if st != N.OK:
            raise AlphaxError(f"{self.lib.axb_status_name(st).decode()}: {self._message()}")
        out = out[: count.value]
        return out.reshape(-1) if k == 1 else out

    def ortho_batch(self, points, r2, eps_singular: float = 1e-12):
        """Device probe of the predicate arithmetic: (m,k,3),(m,k) numpy -> centres, sizes, singular."""
        torch = self.torch
        dev = f"cuda:{self.device}"
        p = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64), device=dev)
        q = torch.as_tensor(np.ascontiguousarray(r2, dtype=np.float64), device=dev)
        m, k = q.shape
        cen = torch.empty((m, 3), dtype=torch.float64, device=dev)
        siz = torch.empty(m, dtype=torch.float64, device=dev)
        sg = torch.zeros(m, dtype=torch.uint8, device=dev)
        with torch.cuda.device(self.device):
            self._bind_stream(fresh=False)
            st = self.lib.axb_ortho_batch(self.handle, m, k, p.data_ptr(), q.data_ptr(), float(eps_singular),
                                          cen.data_ptr(), siz.data_ptr(), sg.data_ptr())
        if st != N.OK:
            raise AlphaxError(self._message())
        return cen.cpu().numpy(), siz.cpu().numpy(), sg.cpu().numpy().astype(bool)


def _max_to_host(a):
    if isinstance(a, np.ndarray):
        return a.max()
    return a.max().item()


_ENGINES: dict = {}


def default_engine(device: int | None = None) -> Engine:
    """Process-wide engine per GPU (keeps the scratch arena warm between calls)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryMissing("CUDA is not available; this package has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    eng = _ENGINES.get(dev)
    if eng is None:
        eng = _ENGINES[dev] = Engine(dev)
    return eng


# --------------------------------------------------------------------------- boundary


def as_ball_arrays(balls: Sequence[Ball]):
    centers = np.array([b.center for b in balls], dtype=np.float64).reshape(-1, 3)
    radii = np.array([b.radius for b in balls], dtype=np.float64)
    return centers, radii


# the keys the reference's compute_alpha_complex writes into stage_times (pipeline.py:498-549, 595)
_REFERENCE_STAGE_KEYS = ("grid", "potential_edges", "potential_triangles", "potential_tets", "prune_tets",
                         "prune_triangles", "prune_edges", "prune_vertices")


def _accumulate_stage_times(stage_times, stage_ms: dict):
    """CUDA-event seconds per stage into the caller's dict -- the reference's keys only (its merge + unique,
    pipeline.py:611-614, is not timed either); the canonicalisation and export times stay in Engine.last_stage_ms."""
    if stage_times is None:
        return
    for key in _REFERENCE_STAGE_KEYS:
        if key in stage_ms:
            stage_times[key] = stage_times.get(key, 0.0) + stage_ms[key] * 1e-3


def compute_alpha_complex_arrays(centers, radii, cfg: PipelineConfig, stage_times: dict | None = None,
                                 device: int | None = None) -> AlphaComplex:
    """Array fast path of ``compute_alpha_complex``: ``centers`` (n,3) and
    ``radii`` (n,) as numpy arrays (ball i = row i).  Same result, no ``Ball``
    objects (building 10^6 of them costs seconds of Python)."""
    if cfg.mode == "naive":
        raise UnsupportedMode("mode='naive' (the reference's exhaustive O(n^4) test oracle, oracle.py) is not part of "
                              "the B200 build; use mode='grid'")
    eng = default_engine(device)
    n = int(np.asarray(radii).shape[0])
    with eng.timing_stages(eng.stage_timing or stage_times is not None):      # events only when somebody reads them
        v, e, t, q = eng.compute_host(centers, radii, cfg)
    if stage_times is not None:
        _accumulate_stage_times(stage_times, eng.last_stage_ms)
    k = AlphaComplex(vertices=v, edges=e, triangles=t, tets=q, alpha=cfg.alpha, ball_count=n)
    # The reference re-checks closure on every result (pipeline.py:623-624).  Here closure holds by construction --
    # a kept simplex marks all its faces on the device, and the emit kernels flag anything inconsistent -- so the
    # host-side re-check (seconds of numpy per million balls) is a debug switch: AXB_CHECK_CLOSURE=1.
    if os.environ.get("AXB_CHECK_CLOSURE") == "1" and not closure_ok(k):
        raise AlphaxError("internal error: output violates closure")
    return k


def compute_alpha_sweep(centers, radii, alphas, cfg: PipelineConfig, device: int | None = None) -> list:
    """``[compute_alpha_complex_arrays(centers, radii, replace(cfg, alpha=a)) for a in alphas]`` with re-use: one
    upload, one grid, one potential stage, one evaluation of every ortho-size and AC2 outcome at max(alphas) (they do
    not depend on alpha), then per alpha only the flags, the inheritance marks and the canonical lists
    (``Engine.sweep_device``).  The complexes are bit-identical to independent runs; if the largest alpha meets a
    singular solve (which a smaller alpha may never evaluate) the sweep falls back to independent runs, so the
    exceptions are the reference's as well."""
    from dataclasses import replace

    import torch

    if cfg.mode == "naive":
        raise UnsupportedMode("mode='naive' is not part of the B200 build; use mode='grid'")
    alphas = [float(a) for a in alphas]
    for a in alphas:
        replace(cfg, alpha=a)                        # the reference's own argument checks, per alpha
    eng = default_engine(device)
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    n = int(radii.shape[0])
    if n == 0:
        raise EmptyInput("at least one ball is required")
    dev = f"cuda:{eng.device}"
    try:
        levels = eng.sweep_device(torch.as_tensor(centers, device=dev), torch.as_tensor(radii, device=dev), alphas, cfg)
    except DegenerateSimplex:
        return [compute_alpha_complex_arrays(centers, radii, replace(cfg, alpha=a), device=device) for a in alphas]
    out = []
    for a, (v, e, t, q) in zip(alphas, levels):
        out.append(AlphaComplex(vertices=v.cpu().numpy(), edges=e.cpu().numpy(), triangles=t.cpu().numpy(),
                                tets=q.cpu().numpy(), alpha=a, ball_count=n))
    return out


def compute_alpha_complex(balls: Sequence[Ball], cfg: PipelineConfig, stage_times: dict | None = None) -> AlphaComplex:
    """Alpha complex of a ball set -- drop-in for the reference entry point
    (pipeline.py:571-628).  ``balls[i].index`` must equal ``i``."""
    if len(balls) == 0:
        raise EmptyInput("at least one ball is required")
    for position, ball in enumerate(balls):
        if ball.index != position:
            raise ValueError(f"ball at position {position} carries index {ball.index}; "
                             "indices must be the stable input ordinals")
    centers, radii = as_ball_arrays(balls)
    return compute_alpha_complex_arrays(centers, radii, cfg, stage_times)
