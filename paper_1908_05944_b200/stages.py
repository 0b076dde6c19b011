"""Standalone stage operations on the GPU -- a "next" row of SURVEY.md 8(f).

Same names and result types as the reference (grid.py:30-62, 91-144;
pipeline.py:86-114, 640-731): ``build_grid``, ``potential_edges``,
``potential_triangles``, ``potential_tets``, ``prune`` with ``Grid``,
``PotentialLevel`` and ``PotentialSets``.  Every call runs the CUDA stages of
the hot path (``axb_grid_build`` / ``axb_potential`` / ``axb_prune`` ...) on the
whole input and exposes the requested intermediate; the cached ortho-centres
and ortho-sizes are the device's fp64 values, bit-identical to the
reference's.  The host only reorders the exported rows into the reference's
canonical (lexicographic) order.

Unlike the reference, a later stage does not consume the Python object of the
previous one -- the device recomputes from the balls -- so passing a hand-edited
level has no effect; the arguments are kept for signature compatibility.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, NamedTuple, Sequence

import numpy as np

from .pipeline import AlphaComplex, PipelineConfig, as_ball_arrays, default_engine
from .types import Ball, OrthoResult, SimplexKey


class CellKey(NamedTuple):
    ix: int
    iy: int
    iz: int


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

    @property
    def ball_count(self) -> int:
        return int(self.order.size)

    def linearize(self, key: CellKey) -> int:
        return key.ix + self.dims[0] * (key.iy + self.dims[1] * key.iz)

    def delinearize(self, linear: int) -> CellKey:
        rest = linear // self.dims[0]
        return CellKey(int(linear % self.dims[0]), int(rest % self.dims[1]), int(rest // self.dims[1]))


@dataclass(frozen=True, eq=False)
class PotentialLevel:
    """Potential simplices of one dimension: rows (m, k) lexicographically sorted, cached
    ortho-centres (m, 3) and ortho-sizes (m,) (reference pipeline.py:86-106)."""

    simplices: np.ndarray
    centers: np.ndarray
    sizes: np.ndarray

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


def _device_inputs(balls: Sequence[Ball]):
    import torch

    centers, radii = as_ball_arrays(balls)
    return torch.as_tensor(centers, device="cuda"), torch.as_tensor(radii, device="cuda")


def build_grid(balls: Sequence[Ball], alpha: float) -> Grid:
    """Uniform grid of side sqrt(r_max^2 + alpha) built by the counting-sort kernels."""
    eng = default_engine()
    dc, dr = _device_inputs(balls)
    info = eng.stage_grid(dc, dr, PipelineConfig(alpha=alpha))
    order, rank, cells = (t.cpu().numpy() for t in eng.stage_grid_export())
    sorted_keys = cells[order]
    change = np.flatnonzero(np.r_[True, sorted_keys[1:] != sorted_keys[:-1]])
    return Grid(origin=info["origin"], cell_side=info["cell_side"], dims=info["dims"], order=order, rank=rank,
                ball_cells=cells, occupied_keys=sorted_keys[change], range_offsets=np.r_[change, order.size].astype(np.int64))


def _level(eng, dim: int) -> PotentialLevel:
    rows, cen, siz = (t.cpu().numpy() for t in eng.stage_potential_export(dim))
    if rows.shape[0]:
        perm = np.lexsort(tuple(rows[:, c] for c in range(rows.shape[1] - 1, -1, -1)))
        rows, cen, siz = rows[perm], cen[perm], siz[perm]
    return PotentialLevel(simplices=rows, centers=cen, sizes=siz)


def _potential(balls: Sequence[Ball], cfg: PipelineConfig, dim: int) -> PotentialLevel:
    eng = default_engine()
    dc, dr = _device_inputs(balls)
    eng.stage_grid(dc, dr, cfg)
    eng.stage_potential()
    return _level(eng, dim)


def potential_edges(grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> PotentialLevel:
    """All edges whose ortho-size is at most alpha + slack (reference pipeline.py:640-646)."""
    return _potential(balls, cfg, 1)


def potential_triangles(edges: PotentialLevel, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> PotentialLevel:
    """Triangles with three potential edges and ortho-size <= alpha + slack (pipeline.py:658-667)."""
    return _potential(balls, cfg, 2)


def potential_tets(triangles: PotentialLevel, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> PotentialLevel:
    """Tetrahedra extending a potential triangle by two more potential edges, ortho-size <= alpha + slack
    (pipeline.py:426-479; the reference's standalone variant pipeline.py:670-709 checks all four faces,
    which is the same set by face monotonicity and is pinned equal by its tests)."""
    return _potential(balls, cfg, 3)


def prune(potentials: PotentialSets, grid: Grid, balls: Sequence[Ball], cfg: PipelineConfig) -> AlphaComplex:
    """Top-down pruning of the whole potential set into the alpha complex (pipeline.py:712-731)."""
    eng = default_engine()
    dc, dr = _device_inputs(balls)
    eng.stage_grid(dc, dr, cfg)
    eng.stage_potential()
    eng.stage_prune()
    counts = eng.stage_canonicalize()
    v, e, t, q = (x.cpu().numpy() for x in eng.stage_export(counts))
    return AlphaComplex(vertices=v, edges=e, triangles=t, tets=q, alpha=cfg.alpha, ball_count=len(balls))
