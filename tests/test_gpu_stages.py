"""The standalone stage API on the GPU against golden cases made with the REAL reference
(tools/make_golden_stages.py: complete and caller-edited levels, AC2 masks, grid queries) and the reference's own
property suites restated for GPU intermediates (reference pkg/tests/test_grid.py:127-171,
pkg/tests/test_pipeline.py:203-249)."""
import json
import os

import numpy as np
import pytest

import oracle
import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import synth

from conftest import GOLD

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stage_cases():
    data = np.load(os.path.join(GOLD, "stage_cases.npz"))
    index = json.load(open(os.path.join(GOLD, "stage_cases.json")))
    return {name: (meta, {k.split("__", 1)[1]: data[k] for k in data.files if k.startswith(name + "__")})
            for name, meta in index.items()}


def balls_of(c, r):
    return [ax.Ball(tuple(float(v) for v in p), float(q), i) for i, (p, q) in enumerate(zip(c, r))]


def thin(level, keep):
    """A level the CALLER made: plain arrays, no device handle."""
    return ax.PotentialLevel(simplices=level.simplices[keep], centers=level.centers[keep], sizes=level.sizes[keep])


def test_stages_consume_complete_and_edited_levels(stage_cases):
    eng = ax.default_engine()
    for name, (meta, a) in stage_cases.items():
        balls = balls_of(a["centers"], a["radii"])
        cfg = ax.PipelineConfig(alpha=meta["alpha"], tolerance=ax.TolerancePolicy(1e-9, meta["eps_singular"]))
        grid = ax.build_grid(balls, meta["alpha"])
        # (1) the chain on device-resident intermediates: nothing is rebuilt between the stages
        token = eng.token
        e = ax.potential_edges(grid, balls, ax.PipelineConfig(alpha=meta["alpha"]))      # default tolerance: same state as build_grid
        assert eng.token == token, "potential_edges rebuilt the grid although its handle was current"
        e = ax.potential_edges(grid, balls, cfg)                                          # another tolerance: rebuilt
        token, edge_id = eng.token, eng.edge_id
        t = ax.potential_triangles(e, grid, balls, cfg)
        q = ax.potential_tets(t, grid, balls, cfg)
        assert eng.token == token and eng.edge_id == edge_id, "a stage re-imported a level whose handle was current"
        for got, want in ((e, a["e"]), (t, a["t"]), (q, a["q"])):
            assert np.array_equal(got.simplices, want.reshape(got.simplices.shape)), name
        for d, lv in ((1, e), (2, t), (3, q)):
            assert np.array_equal(ax.ac2_mask(lv, grid, balls, cfg), a[f"ac2_{d}"]), (name, d)
        k = ax.prune(ax.PotentialSets(edges=e, triangles=t, tets=q, alpha=meta["alpha"]), grid, balls, cfg)
        assert list(k.counts()) == meta["counts_full"]
        for d in range(4):
            assert np.array_equal(k.level(d), a[f"k_full_{d}"].reshape(k.level(d).shape)), (name, d)
        # (2) levels the caller edited are consumed as given -- what the reference's stage functions return for them
        t2 = ax.potential_triangles(thin(e, a["keep_e"]), grid, balls, cfg)
        assert np.array_equal(t2.simplices, a["t_from_e2"]), name
        assert np.array_equal(t2.sizes.view(np.uint64), a["t_from_e2_sizes"].view(np.uint64)), name
        q2 = ax.potential_tets(thin(t, a["keep_t"]), grid, balls, cfg)
        assert np.array_equal(q2.simplices, a["q_from_t2"]), name
        assert np.array_equal(q2.centers.view(np.uint64), a["q_from_t2_centers"].view(np.uint64)), name
        k2 = ax.prune(ax.PotentialSets(edges=e, triangles=t, tets=thin(q, a["keep_q"]), alpha=meta["alpha"]), grid, balls, cfg)
        assert list(k2.counts()) == meta["counts_less_q"]
        for d in range(4):
            assert np.array_equal(k2.level(d), a[f"k_less_q_{d}"].reshape(k2.level(d).shape)), (name, d)
        # AC2 of a hand-made level (rows only) in the caller's order
        perm = np.random.default_rng(1).permutation(len(t))
        shuffled = ax.PotentialLevel(simplices=t.simplices[perm], centers=t.centers[perm], sizes=t.sizes[perm])
        assert np.array_equal(ax.ac2_mask(shuffled, grid, balls, cfg), a["ac2_2"][perm]), name
        # rows that are no simplices of the input are refused, not silently dropped
        bogus = ax.PotentialLevel(simplices=np.array([[0, len(balls) + 5]]), centers=np.zeros((1, 3)), sizes=np.zeros(1))
        with pytest.raises(ax.AlphaxError):
            ax.potential_triangles(bogus, grid, balls, cfg)


def test_grid_queries_against_reference_golden(stage_cases):
    for name, (meta, a) in stage_cases.items():
        balls = balls_of(a["centers"], a["radii"])
        grid = ax.build_grid(balls, meta["alpha"])
        assert np.array_equal(grid.cell_of_array(a["probes"]), a["probe_cells_array"])
        flat, pos = a["neighbors_flat"], 0
        for p, key in zip(a["probes"], a["probe_cells"]):
            assert tuple(ax.cell_of(grid, p)) == tuple(int(v) for v in key)
            for radius in (1, 2):
                m = int(flat[pos])
                want = flat[pos + 1: pos + 1 + m]
                pos += 1 + m
                ck = ax.CellKey(*[int(v) for v in key])
                got = grid.neighbor_indices(ck, radius)
                assert np.array_equal(got, want), (name, key, radius)
                assert list(ax.neighborhood(grid, ck, radius)) == [int(v) for v in want]
        assert pos == len(flat)
        with pytest.raises(ValueError):
            list(ax.neighborhood(grid, ax.CellKey(0, 0, 0), 3))
        ranges = grid.cell_ranges
        assert sum(b - a_ for a_, b in ranges.values()) == len(balls)
        some = next(iter(ranges))
        assert grid.delinearize(grid.linearize(some)) == some


def _ac2_all(centers, r2, level, eps_abs):
    """Domination against ALL balls (the reference's oracle._ac2_all, restated): the locality claim under test is
    that the 27 cells around the ortho-centre are enough."""
    out = np.ones(len(level), dtype=bool)
    for s, (row, c, size) in enumerate(zip(level.simplices, level.centers, level.sizes)):
        d = ((centers - c[None, :]) ** 2).sum(axis=1) - r2
        d[row] = np.inf
        out[s] = not (d < size - eps_abs).any()
    return out


def test_pruning_locality_radius1_equals_all_balls():
    """reference pkg/tests/test_grid.py:127-156 on GPU intermediates."""
    checked = 0
    for seed in range(6):
        c, r = synth.random_globule(70, seed + 100, 1.0, (1.2, 1.9), 1 / 12)
        balls = balls_of(c, r)
        cfg = ax.PipelineConfig(alpha=1.5)
        grid = ax.build_grid(balls, cfg.alpha)
        e = ax.potential_edges(grid, balls, cfg)
        t = ax.potential_triangles(e, grid, balls, cfg)
        q = ax.potential_tets(t, grid, balls, cfg)
        for lv in (e, t, q):
            assert np.array_equal(ax.ac2_mask(lv, grid, balls, cfg), _ac2_all(c, r * r, lv, cfg.tolerance.eps_abs))
            checked += len(lv)
    assert checked > 500


def test_edge_enumeration_completeness_vs_all_pairs():
    """reference pkg/tests/test_grid.py:159-171: the radius-2 enumeration finds exactly the all-pairs set."""
    for seed in (0, 1, 2):
        c, r = synth.random_globule(60, seed + 300, 1.0, (1.2, 1.9), 1 / 12)
        balls = balls_of(c, r)
        cfg = ax.PipelineConfig(alpha=2.0)
        got = ax.potential_edges(ax.build_grid(balls, cfg.alpha), balls, cfg).simplices
        i, j = np.triu_indices(len(balls), 1)
        pts = np.stack([c[i], c[j]], axis=1)
        _, sizes, _ = oracle.ortho_batch(pts, np.stack([r[i] ** 2, r[j] ** 2], axis=1), 1e-12)
        want = np.stack([i, j], axis=1)[sizes <= cfg.alpha + cfg.tolerance.eps_abs]
        assert np.array_equal(got, want)


def test_chunk_ownership_partitions_potentials():
    """reference pkg/tests/test_pipeline.py:203-249: per-chunk potential sets (generators at grid ranks [lo, hi))
    are disjoint, owned by their minimum-rank vertex, and union to the global sets."""
    import torch

    eng = ax.default_engine()
    c, r = synth.random_globule(60, 19, 1.0, (1.2, 1.9), 1 / 12)
    balls = balls_of(c, r)
    cfg = ax.PipelineConfig(alpha=1.5)
    grid = ax.build_grid(balls, cfg.alpha)
    e = ax.potential_edges(grid, balls, cfg)
    t = ax.potential_triangles(e, grid, balls, cfg)
    q = ax.potential_tets(t, grid, balls, cfg)
    n = len(balls)
    parts = {1: [], 2: [], 3: []}
    eng.stage_grid(torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda"), cfg)
    for lo in range(0, n, 13):
        hi = min(lo + 13, n)
        eng.stage_potential(lo, hi)
        for d in (1, 2, 3):
            rows = eng.stage_potential_export(d)[0].cpu().numpy()
            if rows.size:
                min_rank = grid.rank[rows].min(axis=1)
                assert ((min_rank >= lo) & (min_rank < hi)).all()
            parts[d].append(rows)
    for d, level in ((1, e), (2, t), (3, q)):
        stacked = np.concatenate(parts[d], axis=0)
        assert stacked.shape[0] == len(level)                     # disjoint: no duplicates lost
        assert np.array_equal(np.unique(stacked, axis=0), level.simplices)


def test_alpha_sweep_with_reuse_equals_independent_runs():
    """one grid / potential stage / AC2 evaluation at the largest alpha serves every alpha of the
    sweep; each complex must be bit-identical to an independent run (and to the oracle)."""
    cases = [(synth.jittered_lattice(30_000, 21), [0.0, 1.4, 0.3, 0.7, -0.4], False),
             (synth.adversarial_density(20_000, 4, shuffle=True), [0.9, 0.0, 0.45], False),
             (synth.random_globule(2500, 8, 0.5, (0.2, 2.4), 0.12), [1.0, -1.5, 0.0, 0.2, -0.05], False),
             (synth.jittered_lattice(8_000, 22), [0.0, 1.1], True)]
    for (c, r), alphas, bio in cases:
        cfg = ax.PipelineConfig(alpha=0.0, biomolecule_mode=bio, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
        sweep = ax.compute_alpha_sweep(c, r, alphas, cfg)
        assert [k.alpha for k in sweep] == alphas
        for a, k in zip(alphas, sweep):
            from dataclasses import replace

            alone = ax.compute_alpha_complex_arrays(c, r, replace(cfg, alpha=a))
            assert k == alone, (a, k.counts(), alone.counts())
            ref = oracle.compute(c, r, a, eps_singular=1e-300, biomolecule=bio, threads=os.cpu_count(), chunk=2000)
            assert ref.status == oracle.OK
            for got, want in zip((k.vertices, k.edges, k.triangles, k.tets), (ref.vertices, ref.edges, ref.triangles, ref.tets)):
                assert np.array_equal(got, want), a
        for lo, hi in zip(sorted(alphas), sorted(alphas)[1:]):
            assert sweep[alphas.index(lo)].is_subcomplex_of(sweep[alphas.index(hi)])
    # a singular solve at the largest alpha: the sweep falls back to independent runs, i.e. the reference's behaviour
    g = np.stack(np.meshgrid(np.arange(6.0), np.arange(6.0), np.arange(6.0), indexing="ij"), -1).reshape(-1, 3) * 1.5
    with pytest.raises(ax.DegenerateSimplex):
        ax.compute_alpha_sweep(g, np.full(len(g), 1.2), [0.0, 1.0], ax.PipelineConfig(alpha=0.0))


def test_validate_on_the_gpu_path(stage_cases):
    """reference cli.py:134-180: symmetric difference against a partner complex, closure, monotonicity alpha -> alpha+1."""
    meta, a = stage_cases["globule_a1"]
    cfg = ax.PipelineConfig(alpha=meta["alpha"], tolerance=ax.TolerancePolicy(1e-9, meta["eps_singular"]))
    want = ax.AlphaComplex(vertices=a["k_full_0"].reshape(-1), edges=a["k_full_1"], triangles=a["k_full_2"], tets=a["k_full_3"],
                           alpha=meta["alpha"], ball_count=meta["n"])
    rep = ax.validate_complex(a["centers"], a["radii"], cfg, expected=want)
    assert rep.ok and rep.mismatches == (0, 0, 0, 0) and list(rep.counts) == meta["counts_full"]
    assert "closure: ok" in rep.lines()[2] and "monotonicity (alpha -> alpha+1): ok" in rep.lines()[2]
    broken = ax.AlphaComplex(vertices=want.vertices, edges=want.edges[:-3], triangles=want.triangles, tets=want.tets,
                             alpha=want.alpha, ball_count=want.ball_count)
    rep = ax.validate_complex(a["centers"], a["radii"], cfg, expected=broken)
    assert not rep.ok and rep.mismatches[1] == 3 and not rep.closed
    assert ax.validate_complex(a["centers"], a["radii"], ax.PipelineConfig(alpha=0.4)).ok
