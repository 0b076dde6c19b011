"""Standalone stage operations on the GPU -- SURVEY.md 8(f) row 3.

Same names, arguments and result types as the reference (grid.py:30-162;
pipeline.py:86-114, 640-731): ``build_grid``, ``cell_of``, ``neighborhood``,
``potential_edges``, ``potential_triangles``, ``potential_tets``, ``prune``
with ``Grid``, ``PotentialLevel`` and ``PotentialSets``.  Every stage runs the
CUDA kernels of the hot path and, like the reference, CONSUMES what the
previous stage returned:

* a ``Grid`` / ``PotentialLevel`` made here carries an opaque ``device``
  handle.  While the state it names is still resident on the GPU (same
  engine, same balls, same configuration, nothing recomputed since), the next
  stage continues from the device-resident intermediate -- nothing is rebuilt
  or uploaded;
* otherwise (a level the caller built or edited, a stale handle, another
  configuration) the ROWS of the level are uploaded and translated into the
  device layout (``axb_potential_import_edges`` / ``_import_simplices`` /
  ``_tets_from_triangles``), so an edited level has exactly the effect it has
  in the reference.  The cached ortho-centres and ortho-sizes are the device's
  fp64 values, bit-identical to the reference's; ``prune`` recomputes them from
  the rows instead of trusting the arrays of a hand-made level.

The host only reorders exported rows into the reference's canonical
(lexicographic) order.  ``ac2_mask`` exposes pipeline.py:286-313 for one level.
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass, field
from typing import Iterator, NamedTuple, Sequence

import numpy as np

from .errors import EmptyInput
from .pipeline import AlphaComplex, PipelineConfig, as_ball_arrays, default_engine
from .types import Ball, OrthoResult, SimplexKey


class CellKey(NamedTuple):
    ix: int
    iy: int
    iz: int


@dataclass(frozen=True)
class _Handle:
    """Names a device-resident state: engine, run token, fingerprint of (balls, configuration), and which edge /
    simplex level of that run the object describes."""

    engine: object
    token: int
    key: tuple
    edge_id: int = -1
    simplex_id: int = -1


@dataclass(frozen=True, eq=False)
class Grid:
    """Reference grid.py:30-39: geometry, the (cell key, index) order and its inverse,
    per-ball keys, occupied keys and their ranges into ``order``."""

    origin: np.ndarray
    cell_side: float
    dims: tuple
    order: np.ndarray
    rank: np.ndarray
    ball_cells: np.ndarray
    occupied_keys: np.ndarray
    range_offsets: np.ndarray
    device: object = field(default=None, repr=False, compare=False)

    @property
    def ball_count(self) -> int:
        return int(self.order.size)

    def linearize(self, key: CellKey) -> int:
        return key.ix + self.dims[0] * (key.iy + self.dims[1] * key.iz)

    def delinearize(self, linear: int) -> CellKey:
        rest = linear // self.dims[0]
        return CellKey(int(linear % self.dims[0]), int(rest % self.dims[1]), int(rest // self.dims[1]))

    @property
    def cell_ranges(self) -> dict:
        """Occupied cell key -> [start, end) range in ``order`` (grid.py:51-60)."""
        return {self.delinearize(int(k)): (int(a), int(b))
                for k, a, b in zip(self.occupied_keys, self.range_offsets[:-1], self.range_offsets[1:])}

    def cell_of_array(self, points: np.ndarray) -> np.ndarray:
        """Clamped per-axis cell coordinates of points (m, 3) (grid.py:64-67)."""
        q = np.floor((np.asarray(points, dtype=np.float64) - self.origin[None, :]) / self.cell_side).astype(np.int64)
        return np.clip(q, 0, np.asarray(self.dims, dtype=np.int64)[None, :] - 1)

    def neighbor_indices(self, key: CellKey, radius_cells: int) -> np.ndarray:
        """Ball indices of the (2r+1)^3 cell block around ``key`` in ascending (cell key, ball index) order
        (grid.py:69-88).  Walked the way the kernels walk it: consecutive cells of a row are consecutive keys and
        ``order`` is sorted by key, so every (y, z) row of the block is ONE contiguous range of ``order``."""
        dx, dy, dz = self.dims
        x0, x1 = max(0, key.ix - radius_cells), min(dx - 1, key.ix + radius_cells)
        if x0 > x1:
            return np.empty(0, dtype=np.int64)
        parts = []
        for z in range(max(0, key.iz - radius_cells), min(dz - 1, key.iz + radius_cells) + 1):
            for y in range(max(0, key.iy - radius_cells), min(dy - 1, key.iy + radius_cells) + 1):
                row = dx * (y + dy * z)
                a = int(np.searchsorted(self.occupied_keys, row + x0, side="left"))
                b = int(np.searchsorted(self.occupied_keys, row + x1, side="right"))
                if a < b:
                    parts.append(self.order[int(self.range_offsets[a]):int(self.range_offsets[b])])
        if not parts:
            return np.empty(0, dtype=np.int64)
        return parts[0] if len(parts) == 1 else np.concatenate(parts)


def cell_of(grid: Grid, p: Sequence[float]) -> CellKey:
    """Cell containing p, clamped into the grid; a point on a boundary belongs to the higher cell (grid.py:147-153)."""
    q = grid.cell_of_array(np.asarray(p, dtype=np.float64).reshape(1, 3))[0]
    return CellKey(int(q[0]), int(q[1]), int(q[2]))


def neighborhood(grid: Grid, key: CellKey, radius_cells: int) -> Iterator[int]:
    """Every ball whose cell differs from ``key`` by at most ``radius_cells`` per axis (grid.py:156-162)."""
    if radius_cells not in (1, 2):
        raise ValueError("radius_cells must be 1 or 2")
    for idx in grid.neighbor_indices(key, radius_cells):
        yield int(idx)


@dataclass(frozen=True, eq=False)
class PotentialLevel:
    """Potential simplices of one dimension: rows (m, k) lexicographically sorted, cached
    ortho-centres (m, 3) and ortho-sizes (m,) (reference pipeline.py:86-106)."""

    simplices: np.ndarray
    centers: np.ndarray
    sizes: np.ndarray
    device: object = field(default=None, repr=False, compare=False)

    def __len__(self) -> int:
        return int(self.simplices.shape[0])

    def items(self) -> Iterator[tuple]:
        for row, c, s in zip(self.simplices, self.centers, self.sizes):
            yield (SimplexKey(tuple(int(v) for v in row)),
                   OrthoResult(center=tuple(float(x) for x in c), ortho_size=float(s)))


@dataclass(frozen=True, eq=False)
class PotentialSets:
    edges: PotentialLevel
    triangles: PotentialLevel
    tets: PotentialLevel
    alpha: float


# ------------------------------------------------------------------ handles


def _state_key(centers: np.ndarray, radii: np.ndarray, cfg: PipelineConfig) -> tuple:
    return (int(radii.shape[0]), zlib.crc32(centers.tobytes()), zlib.crc32(radii.tobytes()), float(cfg.alpha),
            float(cfg.tolerance.eps_abs), float(cfg.tolerance.eps_singular), bool(cfg.biomolecule_mode))


def _current(handle, eng, key) -> bool:
    return (isinstance(handle, _Handle) and handle.engine is eng and handle.token == eng.token
            and handle.key == key and eng.stage_key == key)


def _ensure_grid(grid, balls: Sequence[Ball], cfg: PipelineConfig, rebuild: bool = False):
    """The engine with the grid of (balls, cfg) resident; rebuilt unless exactly that state is resident already.
    (`grid` is what the caller holds: the reference reads its geometry, here the geometry is a function of
    (balls, cfg.alpha) and is recomputed on the device whenever the resident state is another one.)"""
    if len(balls) == 0:
        raise EmptyInput("at least one ball is required")
    eng = default_engine()
    centers, radii = as_ball_arrays(balls)
    key = _state_key(centers, radii, cfg)
    # (the grid's geometry does not depend on the tolerances, so what decides is whether the state resident on the
    # device was built from these balls under this configuration -- whichever Grid object the caller holds)
    if rebuild or eng.stage_key != key:
        import torch

        eng.stage_grid(torch.as_tensor(centers, device="cuda"), torch.as_tensor(radii, device="cuda"), cfg, key=key)
    return eng, key


def _ensure_edges(edges, grid, balls, cfg):
    """... and with the edge level ``edges`` resident: continued in place when its handle is current, else its rows
    are uploaded (an edited level then has the effect it has in the reference, pipeline.py:658-667)."""
    eng, key = _ensure_grid(grid, balls, cfg)
    h = getattr(edges, "device", None)
    if not (_current(h, eng, key) and h.edge_id == eng.edge_id):
        eng.stage_import_edges(np.asarray(edges.simplices, dtype=np.int64).reshape(-1, 2))
    return eng, key


def _level(eng, dim: int, key) -> PotentialLevel:
    rows, cen, siz = (t.cpu().numpy() for t in eng.stage_potential_export(dim))
    if rows.shape[0]:
        perm = np.lexsort(tuple(rows[:, c] for c in range(rows.shape[1] - 1, -1, -1)))
        rows, cen, siz = rows[perm], cen[perm], siz[perm]
    return PotentialLevel(simplices=rows, centers=cen, sizes=siz,
                          device=_Handle(eng, eng.token, key, eng.edge_id, eng.simplex_id if dim > 1 else -1))


# ------------------------------------------------------------------- stages


def build_grid(balls: Sequence[Ball], alpha: float) -> Grid:
    """Uniform grid of side sqrt(r_max^2 + alpha) built by the counting-sort kernels (grid.py:91-144)."""
    import ctypes as C

    from . import _native as N

    if len(balls) == 0:
        raise EmptyInput("cannot build a grid over zero balls")
    eng, key = _ensure_grid(None, balls, PipelineConfig(alpha=alpha), rebuild=True)
    info = N.GridInfo()
    eng.lib.axb_grid_get_info(eng.handle, C.byref(info))
    order, rank, cells = (t.cpu().numpy() for t in eng.stage_grid_export())
    sorted_keys = cells[order]
    change = np.flatnonzero(np.r_[True, sorted_keys[1:] != sorted_keys[:-1]])
    return Grid(origin=np.array(list(info.origin)), cell_side=float(info.cell_side), dims=tuple(int(d) for d in info.dims),
                order=order, rank=rank, ball_cells=cells, occupied_keys=sorted_keys[change],
                range_offsets=np.r_[change, order.size].astype(np.int64), device=_Handle(eng, eng.token, key))


def potential_edges(grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> PotentialLevel:
    """All edges whose ortho-size is at most alpha + slack (reference pipeline.py:640-646)."""
    eng, key = _ensure_grid(grid, balls, cfg)
    eng.stage_edges()
    return _level(eng, 1, key)


def potential_triangles(edges: PotentialLevel, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> PotentialLevel:
    """Triangles over the GIVEN edges (all three edges in ``edges``) with ortho-size <= alpha + slack
    (pipeline.py:658-667)."""
    eng, key = _ensure_edges(edges, grid, balls, cfg)
    eng.stage_simplices()
    return _level(eng, 2, key)


def potential_tets(triangles: PotentialLevel, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> PotentialLevel:
    """Tetrahedra over the GIVEN triangles: all four faces in ``triangles``, ortho-size <= alpha + slack
    (pipeline.py:670-709).  With a current handle the tets were generated together with the triangles (the hot path
    fuses the two: a potential triangle extended by two more potential edges, pipeline.py:426-479 -- the same set by
    face monotonicity, pinned equal by the reference's tests); otherwise the reference's standalone form runs on the
    uploaded rows."""
    eng, key = _ensure_grid(grid, balls, cfg)
    h = getattr(triangles, "device", None)
    if not (_current(h, eng, key) and h.simplex_id == eng.simplex_id and h.edge_id == eng.edge_id):
        rows = np.asarray(triangles.simplices, dtype=np.int64).reshape(-1, 3)
        if rows.shape[0]:
            perm = np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))
            rows = np.ascontiguousarray(rows[perm])
        # the edge level a tet's partner slots refer to: the edges of the given triangles
        pairs = np.concatenate([rows[:, (0, 1)], rows[:, (0, 2)], rows[:, (1, 2)]], axis=0) if rows.shape[0] else np.empty((0, 2), np.int64)
        eng.stage_import_edges(np.unique(pairs, axis=0) if pairs.shape[0] else pairs)
        eng.stage_tets_from_triangles(rows)
    return _level(eng, 3, key)


def prune(potentials: PotentialSets, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> AlphaComplex:
    """Top-down pruning of the GIVEN potential set into the alpha complex (pipeline.py:712-731)."""
    eng, key = _ensure_grid(grid, balls, cfg)
    he, ht, hq = (getattr(lv, "device", None) for lv in (potentials.edges, potentials.triangles, potentials.tets))
    resident = (all(_current(h, eng, key) for h in (he, ht, hq)) and he.edge_id == ht.edge_id == hq.edge_id == eng.edge_id
                and ht.simplex_id == hq.simplex_id == eng.simplex_id)
    if not resident:
        eng.stage_import_edges(np.asarray(potentials.edges.simplices, dtype=np.int64).reshape(-1, 2))
        eng.stage_import_simplices(np.asarray(potentials.triangles.simplices, dtype=np.int64).reshape(-1, 3),
                                   np.asarray(potentials.tets.simplices, dtype=np.int64).reshape(-1, 4))
    eng.stage_prune()
    counts = eng.stage_canonicalize()
    v, e, t, q = (x.cpu().numpy() for x in eng.stage_export(counts))
    return AlphaComplex(vertices=v, edges=e, triangles=t, tets=q, alpha=cfg.alpha, ball_count=len(balls))


def ac2_mask(level: PotentialLevel, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> np.ndarray:
    """The domination check of the pruning stage for every simplex of ``level`` (pipeline.py:286-313): True where no
    non-incident ball of the 27 cells around the ortho-centre has power distance < size - eps_abs.  Same order as
    ``level.simplices``."""
    dim = int(level.simplices.shape[1]) - 1
    eng, key = _ensure_grid(grid, balls, cfg)
    rows = np.asarray(level.simplices, dtype=np.int64).reshape(-1, dim + 1)
    h = getattr(level, "device", None)
    resident = _current(h, eng, key) and h.edge_id == eng.edge_id and (dim == 1 or h.simplex_id == eng.simplex_id)
    if resident:
        pass                                             # the level is on the device as it is
    elif dim == 1:
        eng.stage_import_edges(rows)
    else:
        pairs = np.concatenate([rows[:, (a, b)] for a in range(dim + 1) for b in range(a + 1, dim + 1)], axis=0)
        eng.stage_import_edges(np.unique(pairs, axis=0) if pairs.shape[0] else pairs.reshape(-1, 2))
        empty3, empty4 = np.empty((0, 3), np.int64), np.empty((0, 4), np.int64)
        eng.stage_import_simplices(rows if dim == 2 else empty3, rows if dim == 3 else empty4)
    got_rows = eng.stage_potential_export(dim)[0].cpu().numpy()
    mask = eng.stage_ac2_mask(dim).cpu().numpy()
    # device order -> the caller's order
    if rows.shape[0] == 0:
        return np.zeros(0, dtype=bool)
    cols = tuple(range(dim, -1, -1))
    back = np.empty(rows.shape[0], dtype=np.int64)
    back[np.lexsort(tuple(rows[:, c] for c in cols))] = np.arange(rows.shape[0])
    return mask[np.lexsort(tuple(got_rows[:, c] for c in cols))][back]
