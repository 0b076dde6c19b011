#!/usr/bin/env python
"""Golden cases for the standalone stage API from the REAL reference package
(build container only: imports ``alphax`` read-only from /root/reference/pkg/src).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_stages.py

For a few seeded instances it records what the reference's own stage functions
return when they are fed the previous stage's level -- complete AND edited
(rows removed by the caller) -- plus the AC2 mask of every level and a few
grid neighbourhood queries:

  potential_triangles(edges', ...)  potential_tets(triangles', ...)  prune(PotentialSets', ...)
  _ac2_mask(level)  Grid.neighbor_indices / cell_of / cell_of_array

-> tests/golden/stage_cases.npz + stage_cases.json.  Test infrastructure only.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import alphax  # noqa: E402  (the reference)
from alphax.grid import CellKey, build_grid, cell_of  # noqa: E402
from alphax.pipeline import PotentialLevel, PotentialSets, _ac2_mask, _NeighborCache, as_ball_arrays  # noqa: E402

from paper_1908_05944_b200 import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def balls_of(centers, radii):
    return [alphax.Ball(tuple(float(v) for v in c), float(r), i) for i, (c, r) in enumerate(zip(centers, radii))]


def thin(level, keep):
    return PotentialLevel(simplices=level.simplices[keep], centers=level.centers[keep], sizes=level.sizes[keep])


def main():
    arrays, index = {}, {}
    cases = [("globule_a1", synth.random_globule(220, 41, 0.9, (1.0, 2.0), 0.07), 1.0),
             ("lattice_a05", synth.jittered_lattice(400, 17), 0.5),
             ("wide_radii_a0", synth.random_globule(180, 5, 0.5, (0.4, 2.3), 0.10), 0.0)]
    for name, (c, r), alpha in cases:
        balls = balls_of(c, r)
        cfg = alphax.PipelineConfig(alpha=alpha, tolerance=alphax.TolerancePolicy(1e-9, 1e-300))
        grid = build_grid(balls, alpha)
        centers, radii = as_ball_arrays(balls)
        r2 = radii * radii
        e = alphax.potential_edges(grid, balls, cfg)
        t = alphax.potential_triangles(e, grid, balls, cfg)
        q = alphax.potential_tets(t, grid, balls, cfg)
        rng = np.random.default_rng(len(balls))
        keep_e = rng.random(len(e)) > 0.15
        keep_t = rng.random(len(t)) > 0.15
        keep_q = rng.random(len(q)) > 0.30
        e2, t2 = thin(e, keep_e), thin(t, keep_t)
        t_from_e2 = alphax.potential_triangles(e2, grid, balls, cfg)
        q_from_t2 = alphax.potential_tets(t2, grid, balls, cfg)
        k_full = alphax.prune(PotentialSets(edges=e, triangles=t, tets=q, alpha=alpha), grid, balls, cfg)
        # an edited but still closed potential set: fewer tets, everything else complete
        k_less_q = alphax.prune(PotentialSets(edges=e, triangles=t, tets=thin(q, keep_q), alpha=alpha), grid, balls, cfg)
        rec = dict(n=len(balls), alpha=alpha, eps_singular=1e-300, counts_full=list(k_full.counts()),
                   counts_less_q=list(k_less_q.counts()))
        put = {"centers": c, "radii": r, "e": e.simplices, "t": t.simplices, "q": q.simplices,
               "keep_e": keep_e, "keep_t": keep_t, "keep_q": keep_q,
               "t_from_e2": t_from_e2.simplices, "t_from_e2_sizes": t_from_e2.sizes,
               "q_from_t2": q_from_t2.simplices, "q_from_t2_centers": q_from_t2.centers}
        for d, lv in ((1, e), (2, t), (3, q)):
            put[f"ac2_{d}"] = _ac2_mask(centers, r2, grid, _NeighborCache(grid), lv.simplices, lv.centers, lv.sizes,
                                        cfg.tolerance.eps_abs)
        for tag, k in (("full", k_full), ("less_q", k_less_q)):
            for d in range(4):
                put[f"k_{tag}_{d}"] = k.level(d)
        # grid queries
        probes = rng.uniform(c.min(axis=0) - 1.0, c.max(axis=0) + 1.0, size=(12, 3))
        probes[0] = grid.origin                                     # on the lower corner
        probes[1] = grid.origin + grid.cell_side * np.array([1.0, 2.0, 0.0])   # exactly on cell boundaries
        put["probes"] = probes
        put["probe_cells"] = np.array([tuple(cell_of(grid, p)) for p in probes], dtype=np.int64)
        put["probe_cells_array"] = grid.cell_of_array(probes)
        nb = []
        for p, key in zip(probes, put["probe_cells"]):
            for radius in (1, 2):
                got = grid.neighbor_indices(CellKey(*[int(v) for v in key]), radius)
                nb.append(np.r_[len(got), got])
        put["neighbors_flat"] = np.concatenate(nb).astype(np.int64)
        for k, v in put.items():
            arrays[f"{name}__{k}"] = np.asarray(v)
        index[name] = rec
        print(name, rec, len(e), len(t), len(q), "->", len(t_from_e2), len(q_from_t2))
    np.savez_compressed(os.path.join(GOLD, "stage_cases.npz"), **arrays)
    json.dump(index, open(os.path.join(GOLD, "stage_cases.json"), "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
