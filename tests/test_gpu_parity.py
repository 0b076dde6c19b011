"""GPU parity tests: the CUDA path (through the Python boundary and the C-ABI)
against (a) the golden outputs of the real reference and (b) the CPU oracle on
the same seeded inputs.  Bit-exact everywhere: integer rows and the cached
fp64 ortho data."""
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import synth

from conftest import GOLD
from helpers import canonical_text, digest_arrays, digest_values

pytestmark = pytest.mark.gpu


def arrays_of(k):
    return (k.vertices, k.edges, k.triangles, k.tets)


def assert_same_complex(k, ref, tag=""):
    for d, (got, want) in enumerate(zip(arrays_of(k), (ref.vertices, ref.edges, ref.triangles, ref.tets))):
        assert got.dtype == np.int64
        assert np.array_equal(got, want), f"{tag}: dimension {d} differs"


def lexsorted(rows, *carry):
    if rows.shape[0] == 0:
        return (rows,) + carry
    perm = np.lexsort(tuple(rows[:, c] for c in range(rows.shape[1] - 1, -1, -1)))
    return (rows[perm],) + tuple(a[perm] for a in carry)


def test_device_ortho_matches_reference_bitwise():
    eng = ax.default_engine()
    d = np.load(os.path.join(GOLD, "ortho_vectors.npz"))
    for k in (1, 2, 3, 4):
        for eps in ("1e-12", "1e-300"):
            cen, siz, sg = eng.ortho_batch(d[f"k{k}_points"], d[f"k{k}_r2"], float(eps))
            want_sg = d[f"k{k}_eps{eps}_singular"]
            assert np.array_equal(sg, want_sg)
            ok = ~want_sg
            assert np.array_equal(cen[ok].view(np.uint64), d[f"k{k}_eps{eps}_centers"][ok].view(np.uint64))
            assert np.array_equal(siz[ok].view(np.uint64), d[f"k{k}_eps{eps}_sizes"][ok].view(np.uint64))


def test_small_cases_against_reference_golden(gold_small):
    for name, rec in gold_small.items():
        m = rec["meta"]
        cfg = ax.PipelineConfig(alpha=m["alpha"], biomolecule_mode=m["biomolecule"],
                                tolerance=ax.TolerancePolicy(m["eps_abs"], m["eps_singular"]))
        k = ax.compute_alpha_complex_arrays(rec["centers"], rec["radii"], cfg)
        assert list(k.counts()) == m["counts"], name
        for d, got in enumerate(arrays_of(k)):
            assert np.array_equal(got, rec[f"k{d}"].reshape(got.shape)), (name, d)
        text = canonical_text(*arrays_of(k), len(rec["radii"]), m["alpha"])
        assert hashlib.sha256(text.encode()).hexdigest() == m["sha256_complex"], name
        assert k.ball_count == len(rec["radii"]) and k.alpha == m["alpha"]


def test_config1_through_ball_boundary(gold_config1):
    data, meta = gold_config1
    balls = [ax.Ball(tuple(c), float(r), i) for i, (c, r) in enumerate(zip(data["centers"], data["radii"]))]
    for tag, m in meta.items():
        st = {}
        k = ax.compute_alpha_complex(balls, ax.PipelineConfig(alpha=m["alpha"], biomolecule_mode=m["biomolecule"],
                                                              workers=3, chunk_size=37), stage_times=st)
        assert list(k.counts()) == m["counts"]
        for d, got in enumerate(arrays_of(k)):
            assert np.array_equal(got, data[f"{tag}__k{d}"].reshape(got.shape))
        text = canonical_text(*arrays_of(k), 1000, m["alpha"])
        assert hashlib.sha256(text.encode()).hexdigest() == m["sha256_complex"]
        for key in ("grid", "potential_edges", "potential_triangles", "potential_tets", "prune_tets",
                    "prune_triangles", "prune_edges", "prune_vertices"):
            assert key in st and st[key] >= 0.0
        assert ax.closure_ok(k)
        assert ax.complex_stats(k).total == sum(m["counts"])


def test_stage_times_are_recorded_on_request_only():
    """The reference fills `stage_times` only for a caller who passes a dict (pipeline.py:571, 595); here the CUDA
    events behind it are recorded only then (axb_set_stage_timing): same complex either way."""
    c, r = synth.jittered_lattice(20_000, seed=5)
    cfg = ax.PipelineConfig(alpha=0.4)
    eng = ax.default_engine()
    assert not eng.stage_timing
    plain = ax.compute_alpha_complex_arrays(c, r, cfg)
    assert sum(eng.last_stage_ms.values()) == 0.0
    st = {}
    timed = ax.compute_alpha_complex_arrays(c, r, cfg, stage_times=st)
    assert not eng.stage_timing                                   # restored
    assert st["potential_edges"] > 0.0 and st["prune_triangles"] > 0.0 and st["grid"] > 0.0
    for a, b in zip(arrays_of(plain), arrays_of(timed)):
        assert np.array_equal(a, b)
    import torch
    dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
    with eng.timing_stages():
        eng.compute_device(dc, dr, cfg)
        assert eng.last_stage_ms["potential_triangles"] > 0.0 and eng.last_stage_ms["canonical"] > 0.0
    eng.compute_device(dc, dr, cfg)
    assert sum(eng.last_stage_ms.values()) == 0.0


def test_stagewise_against_oracle():
    """grid order, potential levels (rows + cached ortho data bitwise) and the complex, stage by stage."""
    import torch

    eng = ax.default_engine()
    cases = [synth.jittered_lattice(20_000, 11) + (0.0, 1e-12), synth.jittered_lattice(20_000, 11) + (1.4, 1e-12),
             synth.adversarial_density(20_000, 5) + (0.0, 1e-300),
             synth.random_globule(300, 21, 0.4, (0.3, 2.2), 0.5) + (0.7, 1e-300)]
    for c, r, alpha, eps_sing in cases:
        cfg = ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps_sing))
        ref = oracle.compute(c, r, alpha, eps_singular=eps_sing, keep_potentials=True, threads=os.cpu_count(), chunk=2000)
        assert ref.status == oracle.OK
        info = eng.stage_grid(torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda"), cfg)
        st, g = oracle.grid_build(c, r, alpha)
        assert info["dims"] == g.dims and info["cell_side"] == g.side and np.array_equal(info["origin"], g.origin)
        order, rank, cells = (t.cpu().numpy() for t in eng.stage_grid_export())
        assert np.array_equal(order, g.order) and np.array_equal(rank, g.rank) and np.array_equal(cells, g.cells)
        eng.stage_potential()
        for dim in (1, 2, 3):
            rows, cen, siz = lexsorted(*(t.cpu().numpy() for t in eng.stage_potential_export(dim)))
            wrows, wcen, wsiz = ref.potentials[dim]
            assert np.array_equal(rows, wrows), dim
            assert np.array_equal(cen.view(np.uint64), wcen.view(np.uint64)), dim
            assert np.array_equal(siz.view(np.uint64), wsiz.view(np.uint64)), dim
        eng.stage_prune()
        counts = eng.stage_canonicalize()
        outs = [t.cpu().numpy() for t in eng.stage_export(counts)]
        for got, want in zip(outs, (ref.vertices, ref.edges, ref.triangles, ref.tets)):
            assert np.array_equal(got, want)


def test_error_parity(gold_errors):
    """Same exception type, vertices and message as the reference on its failing inputs."""
    kinds = {"DegenerateSimplex": ax.DegenerateSimplex, "DuplicateCenter": ax.DuplicateCenter,
             "NonFiniteCoordinate": ax.NonFiniteCoordinate, "ValueError": ValueError}
    for name, rec in gold_errors.items():
        c = np.array(rec["centers"], dtype=np.float64)
        r = np.array(rec["radii"], dtype=np.float64)
        cfg = ax.PipelineConfig(alpha=rec["alpha"], tolerance=ax.TolerancePolicy(1e-9, rec["eps_singular"]))
        if rec["error"] is None:
            ax.compute_alpha_complex_arrays(c, r, cfg)
            continue
        with pytest.raises(kinds[rec["error"]]) as err:
            ax.compute_alpha_complex_arrays(c, r, cfg)
        assert str(err.value) == rec["message"], name
        if rec["error"] == "DegenerateSimplex":
            assert list(err.value.vertices) == rec["vertices"], name
    with pytest.raises(ax.EmptyInput):
        ax.compute_alpha_complex([], ax.PipelineConfig(alpha=0.0))
    with pytest.raises(ax.NonFiniteCoordinate, match="ball 1 is not finite"):
        ax.compute_alpha_complex_arrays(np.array([[0, 0, 0], [np.inf, 0, 0]]), np.ones(2), ax.PipelineConfig(alpha=0.0))
    with pytest.raises(ValueError, match="stable input ordinals"):
        ax.compute_alpha_complex([ax.Ball((0, 0, 0), 1, 0), ax.Ball((3, 0, 0), 1, 2)], ax.PipelineConfig(alpha=0.0))
    with pytest.raises(NotImplementedError):
        ax.compute_alpha_complex_arrays(np.zeros((1, 3)), np.ones(1), ax.PipelineConfig(alpha=0.0, mode="naive"))


def test_many_singular_solves_report_the_first():
    """More singular candidates than record slots: the replay path must still name the reference's simplex."""
    g = np.stack(np.meshgrid(np.arange(14.0), np.arange(14.0), np.arange(14.0), indexing="ij"), -1).reshape(-1, 3) * 1.5
    r = np.full(g.shape[0], 1.2)
    ref = oracle.compute(g, r, 1.0)
    assert ref.status == oracle.DEGENERATE
    with pytest.raises(ax.DegenerateSimplex) as err:
        ax.compute_alpha_complex_arrays(g, r, ax.PipelineConfig(alpha=1.0))
    assert err.value.vertices == ref.error_vertices


def test_config2_50k_against_reference_golden(gold_large):
    for name in ("g2_50k_a0", "g2_50k_a14"):
        m = gold_large[name]
        c, r = synth.jittered_lattice(m["n"], m["seed"])
        k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=m["alpha"]))
        assert list(k.counts()) == m["counts"]
        assert digest_arrays(*arrays_of(k)) == m["sha256_arrays"]
    # alpha sweep is monotone: K(0) is a subcomplex of K(1.4)
    c, r = synth.jittered_lattice(20_000, 0)
    k0 = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=0.0))
    k1 = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=1.4))
    assert k0.is_subcomplex_of(k1) and ax.closure_ok(k0) and ax.closure_ok(k1)


def test_config3_1m_against_oracle_and_reference_golden(gold_large):
    """1,000,000 atoms, alpha 0 -- full-size bit-exact comparison."""
    c, r = synth.jittered_lattice(1_000_000, 0)
    k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=0.0))
    assert k.counts() == (1000000, 4607698, 3483769, 510141)          # measured with the reference
    if "g2_1m_a0" in gold_large:
        assert list(k.counts()) == gold_large["g2_1m_a0"]["counts"]
        assert digest_arrays(*arrays_of(k)) == gold_large["g2_1m_a0"]["sha256_arrays"]
    ref = oracle.compute(c, r, 0.0, threads=os.cpu_count(), chunk=4000)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "1M")
    # rows strictly increasing and lexicographically sorted without duplicates (size-independent properties)
    for rows in (k.edges, k.triangles, k.tets):
        assert (np.diff(rows, axis=1) > 0).all()
        a, b = rows[:-1], rows[1:]
        less = np.zeros(a.shape[0], dtype=bool)
        equal = np.ones(a.shape[0], dtype=bool)
        for col in range(rows.shape[1]):
            less |= equal & (a[:, col] < b[:, col])
            equal &= a[:, col] == b[:, col]
        assert less.all()
    assert (np.diff(k.vertices) > 0).all()


def test_config3_1m_alpha14_against_oracle_and_survey_counts():
    """SURVEY.md 8(d) config 3 at alpha = 1.4 with the H1 pivot threshold (1e-300): the counts the survey measured
    with the real reference, and every row against the CPU oracle."""
    c, r = synth.jittered_lattice(1_000_000, 0)
    tol = ax.TolerancePolicy(1e-9, 1e-300)
    k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=1.4, tolerance=tol))
    assert k.counts() == (1000000, 7245190, 11673237, 5174354)
    ref = oracle.compute(c, r, 1.4, eps_singular=1e-300, threads=os.cpu_count(), chunk=4000)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "1M a1.4")
    # with the default threshold both sides raise on the tet the survey names
    with pytest.raises(ax.DegenerateSimplex) as err:
        ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=1.4))
    assert tuple(err.value.vertices) == (236991, 237091, 246991, 247091)


def test_config5_adversarial_1m_against_oracle():
    """BASELINE config 5 at full size: 1M atoms, 20 % of the volume carved into voids, 20 % of the atoms in 3x-dense
    cores, alpha 0, H1 tolerance -- no golden exists, the oracle is computed in the same run."""
    c, r = synth.adversarial_density(1_000_000, 0)
    tol = ax.TolerancePolicy(1e-9, 1e-300)
    k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=0.0, tolerance=tol))
    ref = oracle.compute(c, r, 0.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=4000)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "adversarial 1M")
    assert ax.closure_ok(k)


def test_config4_10m_on_one_gpu_counts_and_oracle():
    """BASELINE config 4's input (10M atoms, alpha 0, H1 tolerance) in ONE pass on one GPU: the counts the builder
    logged against the oracle in round 1, every row against the oracle again, and the size-independent properties."""
    c, r = synth.jittered_lattice(10_000_000, 0)
    tol = ax.TolerancePolicy(1e-9, 1e-300)
    k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=0.0, tolerance=tol))
    assert k.counts() == (10000000, 46142433, 34798584, 5092246)
    for rows in (k.edges, k.triangles, k.tets):
        assert (np.diff(rows, axis=1) > 0).all()
        a, b = rows[:-1], rows[1:]
        less = np.zeros(a.shape[0], dtype=bool)
        equal = np.ones(a.shape[0], dtype=bool)
        for col in range(rows.shape[1]):
            less |= equal & (a[:, col] < b[:, col])
            equal &= a[:, col] == b[:, col]
        assert less.all()
    ref = oracle.compute(c, r, 0.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=8000)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "10M")


def test_alpha14_200k_tiny_eps_against_oracle():
    c, r = synth.jittered_lattice(200_000, 0)
    tol = ax.TolerancePolicy(1e-9, 1e-300)
    k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=1.4, tolerance=tol))
    ref = oracle.compute(c, r, 1.4, eps_singular=1e-300, threads=os.cpu_count(), chunk=4000)
    assert_same_complex(k, ref, "200k a1.4")


def test_adversarial_density_against_oracle():
    """Config 5 (reduced to 300k atoms so the CPU oracle stays quick): voids + 3x-dense cores, shuffled indices."""
    c, r = synth.adversarial_density(300_000, 0, shuffle=True)
    tol = ax.TolerancePolicy(1e-9, 1e-300)
    k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=0.0, tolerance=tol))
    ref = oracle.compute(c, r, 0.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=4000)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "adversarial")


def test_dense_blob_crowded_edge_batches_against_oracle():
    """~60 potential-edge partners per ball: a warp batch of 8 generators overflows its pair queue, so
    k_edges has to halve batches (and k_tri_tet3 runs its wide W=4 variant)."""
    rng = np.random.default_rng(11)
    c = rng.uniform(0.0, 11.0, size=(500, 3))
    r = rng.uniform(1.2, 1.9, size=500)
    tol = ax.TolerancePolicy(1e-9, 1e-300)
    for alpha in (1.0, 0.0):
        k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=alpha, tolerance=tol))
        ref = oracle.compute(c, r, alpha, eps_singular=1e-300, threads=os.cpu_count(), chunk=16)
        assert ref.status == oracle.OK
        assert_same_complex(k, ref, f"dense blob alpha={alpha}")


def test_hundreds_of_partners_per_ball_against_oracle():
    """The reference has no density limit (pipeline.py:316-359).  alpha = 40 A^2 at protein density gives every
    ball several hundred potential-edge partners: more than the pair queue of k_edges (two-sweep path), more than
    a k_tri_tet3 tile (heavy.cuh: bit matrices in global scratch) and a kept-triangle mask of 5+ words per row."""
    import torch

    tol = ax.TolerancePolicy(1e-9, 1e-300)
    c, r = synth.jittered_lattice(700, 31)
    k = ax.compute_alpha_complex_arrays(c[:450], r[:450], ax.PipelineConfig(alpha=40.0, tolerance=tol))
    ref = oracle.compute(c[:450], r[:450], 40.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=16)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "alpha=40")
    # (this input does take the heavy paths: potential edges = all pairs with ortho-size <= alpha + slack, the
    # completeness property of reference pkg/tests/test_grid.py:159-171; partners are counted at the lower grid rank)
    i, j = np.triu_indices(450, 1)
    _, sizes, _ = oracle.ortho_batch(np.stack([c[i], c[j]], axis=1), np.stack([r[i] ** 2, r[j] ** 2], axis=1), 1e-300)
    pot = sizes <= 40.0 + 1e-9
    st, g = oracle.grid_build(c[:450], r[:450], 40.0)
    assert np.bincount(np.minimum(g.rank[i[pot]], g.rank[j[pot]])).max() > 300
    # the stage API sees the same potential levels (complete lists: no cull) at up to 256 partners per generator
    eng = ax.default_engine()
    cfg = ax.PipelineConfig(alpha=40.0, tolerance=tol)
    c3, r3 = c[:300], r[:300]
    ref = oracle.compute(c3, r3, 40.0, eps_singular=1e-300, keep_potentials=True, threads=os.cpu_count(), chunk=16)
    eng.stage_grid(torch.as_tensor(c3, device="cuda"), torch.as_tensor(r3, device="cuda"), cfg, arena_factor=64.0)
    eng.stage_potential()
    for dim in (1, 2, 3):
        rows = lexsorted(eng.stage_potential_export(dim)[0].cpu().numpy())[0]
        assert np.array_equal(rows, ref.potentials[dim][0]), dim
    # a dense blob in a sparse surrounding: only a few generators take the heavy path
    rng = np.random.default_rng(5)
    blob = rng.uniform(0.0, 9.0, size=(420, 3)) + 20.0
    c2 = np.concatenate([synth.jittered_lattice(3000, 2)[0], blob])
    r2 = rng.uniform(1.2, 1.9, size=len(c2))
    k = ax.compute_alpha_complex_arrays(c2, r2, ax.PipelineConfig(alpha=6.0, tolerance=tol))
    ref = oracle.compute(c2, r2, 6.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=16)
    assert ref.status == oracle.OK
    assert_same_complex(k, ref, "dense blob in a lattice")
    # 620 balls strung along a 2.9 A arc of a 50 A circle: every pair is a potential edge (up to 604 partners per
    # generator, more than the pair queue of k_edges holds: its two-sweep path; kept-triangle mask of 10 words per row)
    n, rho = 620, 50.0
    th = np.linspace(0.0, 2.9 / rho, n)
    arc = np.stack([rho * np.cos(th), rho * np.sin(th), rng.uniform(-3e-3, 3e-3, size=n)], axis=1)[rng.permutation(n)]
    ra = rng.uniform(1.45, 1.55, size=n)
    for bio in (False, True):
        k = ax.compute_alpha_complex_arrays(arc, ra, ax.PipelineConfig(alpha=0.0, biomolecule_mode=bio, tolerance=tol))
        ref = oracle.compute(arc, ra, 0.0, eps_singular=1e-300, biomolecule=bio, keep_potentials=True, threads=os.cpu_count(), chunk=16)
        assert ref.status == oracle.OK and len(ref.edges) > 0
        assert_same_complex(k, ref, "balls on an arc")
    st, g = oracle.grid_build(arc, ra, 0.0)
    assert np.bincount(g.rank[ref.potentials[1][0]].min(axis=1)).max() > 500
    # flatter (z within 1e-4 A): four balls turn out affinely dependent to the last bit; the heavy path must name the
    # tetrahedron the reference meets first in its enumeration
    flat = arc.copy()
    flat[:, 2] = rng.uniform(-1e-4, 1e-4, size=n)
    bad = oracle.compute(flat, ra, 0.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=16)
    if bad.status == oracle.DEGENERATE:
        with pytest.raises(ax.DegenerateSimplex) as err:
            ax.compute_alpha_complex_arrays(flat, ra, ax.PipelineConfig(alpha=0.0, tolerance=tol))
        assert tuple(err.value.vertices) == tuple(bad.error_vertices)
    eng.stage_grid(torch.as_tensor(arc, device="cuda"), torch.as_tensor(ra, device="cuda"), ax.PipelineConfig(alpha=0.0, tolerance=tol), arena_factor=64.0)
    eng.stage_potential()
    for dim in (1, 2, 3):
        rows = lexsorted(eng.stage_potential_export(dim)[0].cpu().numpy())[0]
        assert np.array_equal(rows, ref.potentials[dim][0]), dim


def test_randomised_shapes_against_oracle():
    """tools/gpu_fuzz.py as a test: 120 small inputs of many shapes (clusters, near-lattices with ties, far-away
    offsets, flat slabs, lines; wide radii, negative alpha, both vertex modes, both pivot thresholds): same
    arrays, and the same DegenerateSimplex vertices where the reference raises."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("gpu_fuzz", os.path.join(os.path.dirname(GOLD), "..", "tools", "gpu_fuzz.py"))
    fuzz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fuzz)
    rng = np.random.default_rng(12345)
    raised = 0
    for i in range(120):
        c, r, alpha, bio, eps_sing = fuzz.make_case(rng)
        ref = oracle.compute(c, r, alpha, eps_singular=eps_sing, biomolecule=bio, threads=4, chunk=64)
        cfg = ax.PipelineConfig(alpha=alpha, biomolecule_mode=bio, tolerance=ax.TolerancePolicy(1e-9, eps_sing))
        if ref.status == oracle.DEGENERATE:
            raised += 1
            with pytest.raises(ax.DegenerateSimplex) as info:
                ax.compute_alpha_complex_arrays(c, r, cfg)
            assert tuple(info.value.vertices) == tuple(ref.error_vertices), f"case {i}"
        else:
            assert ref.status == oracle.OK
            assert_same_complex(ax.compute_alpha_complex_arrays(c, r, cfg), ref, f"fuzz case {i}")


def test_optimistic_list_sizes_are_redone_when_they_do_not_hold(monkeypatch):
    """axb_compute sizes the potential-tet list by a guess and checks it only at the end (no host round trip after
    the triangle/tet kernel); AXB_TEST_SMALL_PQ makes the guess fail so the redo path (and the host path's
    retry loop) must produce the same complex."""
    import torch

    eng = ax.default_engine()
    c, r = synth.jittered_lattice(60_000, 4)
    cfg = ax.PipelineConfig(alpha=1.0)
    want = eng.compute_host(c, r, cfg)
    monkeypatch.setenv("AXB_TEST_SMALL_PQ", "1")
    eng.arena.fill_(0x7F)
    dev = [t.cpu().numpy() for t in eng.compute_device(torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda"), cfg)]
    host = eng.compute_host(c, r, cfg)
    for a, b, h in zip(want, dev, host):
        assert np.array_equal(a, b) and np.array_equal(a, h)


def test_remembered_sizes_are_verified_and_redone():
    """The device path remembers list lengths per problem shape (n, configuration, grid dims) and, on the next call with
    that shape, neither waits for the edge counters nor for the row counts before it emits.  A different point set of the
    same shape must still come out right: denser interior (more partners than remembered -> the run is redone exactly),
    and a sparser one (the remembered sizes hold)."""
    import torch

    eng = ax.default_engine()
    c, r = synth.jittered_lattice(30_000, 14)
    r = r.copy()
    r[0] = 1.9                                          # the same r_max, hence the same cell side, in every variant
    mid = 0.5 * (c.min(axis=0) + c.max(axis=0))
    keep = np.unique(np.concatenate([c.argmin(axis=0), c.argmax(axis=0)]))      # the balls that span the bounding box

    def variant(scale):
        v = mid + (c - mid) * scale
        v[keep] = c[keep]
        return np.ascontiguousarray(v)

    cfg = ax.PipelineConfig(alpha=0.3, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
    launches = []
    for scale in (1.0, 1.0, 0.8, 0.8, 1.15, 1.0):
        v = variant(scale)
        want = eng.compute_host(v, r, cfg)
        eng.arena.fill_(0x7F)            # whatever a run on remembered sizes leaves unwritten must not be read either
        before = eng.kernel_launches
        got = [t.cpu().numpy() for t in eng.compute_device(torch.as_tensor(v, device="cuda"), torch.as_tensor(r, device="cuda"), cfg)]
        launches.append(eng.kernel_launches - before)
        for a, b in zip(want, got):
            assert a.dtype == b.dtype == np.int64 and np.array_equal(a, b), scale
    # the second call ran once (remembered sizes held), the third had to be redone (about twice the launches)
    assert launches[2] > launches[1] + 8 and launches[3] <= launches[1] + 2


def test_device_path_equals_host_path_and_is_deterministic():
    import torch

    eng = ax.default_engine()
    c, r = synth.jittered_lattice(100_000, 2)
    cfg = ax.PipelineConfig(alpha=0.5)
    host = eng.compute_host(c, r, cfg)
    for _ in range(2):
        dev = [t.cpu().numpy() for t in eng.compute_device(torch.as_tensor(c, device="cuda"),
                                                           torch.as_tensor(r, device="cuda"), cfg)]
        for a, b in zip(host, dev):
            assert np.array_equal(a, b)
    before = eng.kernel_launches
    eng.compute_host(c, r, cfg)
    assert eng.kernel_launches - before >= 20        # the CUDA kernels did run


def test_permutation_of_input_indices():
    """Relabelling the balls relabels the complex (ownership by grid rank must not leak into the output)."""
    c, r = synth.jittered_lattice(30_000, 4)
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(r))
    cfg = ax.PipelineConfig(alpha=0.8)
    k = ax.compute_alpha_complex_arrays(c, r, cfg)
    kp = ax.compute_alpha_complex_arrays(c[perm], r[perm], cfg)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    # ball i of the original is ball inv[i] of the permuted input
    relabelled = ax.AlphaComplex.from_rows(inv[k.vertices], np.sort(inv[k.edges], axis=1),
                                           np.sort(inv[k.triangles], axis=1), np.sort(inv[k.tets], axis=1),
                                           cfg.alpha, len(r))
    assert relabelled == kp


def test_slab_sharding_on_one_gpu_equals_single_shot():
    """All slabs of a 3- and 8-way sharded run computed one after the other on this GPU: every slab must emit
    exactly the simplices of the complex whose generator (minimum grid rank vertex) it owns -- inherited faces
    decided from its lower halo included -- so the lists are disjoint, add up to the global counts, and their
    merge equals the unsharded result bit for bit."""
    from paper_1908_05944_b200 import sharding
    from helpers import rows_generated_in

    eng = ax.default_engine()
    for (c, r), alpha, eps, bio in ((synth.jittered_lattice(60_000, 8), 0.0, 1e-12, False),
                                    (synth.jittered_lattice(30_000, 8), 1.4, 1e-300, False),
                                    (synth.adversarial_density(30_000, 3, shuffle=True), 0.0, 1e-300, False),
                                    (synth.random_globule(3000, 5, 0.5, (0.2, 2.4), 0.12), 0.3, 1e-300, False),
                                    (synth.jittered_lattice(20_000, 2), 0.6, 1e-300, True)):
        cfg = ax.PipelineConfig(alpha=alpha, biomolecule_mode=bio, tolerance=ax.TolerancePolicy(1e-9, eps))
        single = eng.compute_host(c, r, cfg)
        st, g = oracle.grid_build(c, r, alpha)
        for world in (3, 8):
            merged, per_rank = sharding.compute_sharded_single_gpu(c, r, cfg, world, eng)
            plan = sharding.plan_slabs(c, r, alpha, world)
            for d in range(4):
                assert np.array_equal(merged[d].cpu().numpy(), single[d]), (world, d)
                assert sum(int(o[d].shape[0]) for o in per_rank) == single[d].shape[0], (world, d)   # disjoint
            for rank, outs in enumerate(per_rank):
                want = rows_generated_in(single, g.rank, *plan.rank_ranges[rank])
                for d in range(4):
                    assert np.array_equal(outs[d].cpu().numpy(), want[d]), (world, rank, d)


def test_slab_errors_name_global_balls():
    """A slab that meets a singular solve or a duplicate centre reports GLOBAL ball indices and the detail the
    ranks of a sharded run need to agree on the error the reference raises for the whole input."""
    import torch

    from paper_1908_05944_b200 import sharding

    eng = ax.default_engine()
    c, r = synth.jittered_lattice(20_000, 3)
    # (a) duplicate centre far up the z axis
    top = np.argsort(c[:, 2])[-40:]
    c_dup = c.copy()
    i, j = sorted((int(top[3]), int(top[17])))
    c_dup[j] = c_dup[i]
    cfg = ax.PipelineConfig(alpha=0.0)
    with pytest.raises(ax.DuplicateCenter) as whole:
        ax.compute_alpha_complex_arrays(c_dup, r, cfg)
    jobs = [sharding.ShardedJob(c_dup, r, cfg, q, 4, eng) for q in range(4)]
    errs = [job.local(raise_errors=False)[1] for job in jobs]
    assert errs[0] is None and errs[3] is not None and errs[3].vertices == (i, j)
    hit = sharding.pick_error(errs)
    with pytest.raises(ax.DuplicateCenter) as sharded:
        eng.raise_slab_error(hit[1], cfg)
    assert str(sharded.value) == str(whole.value)
    # (b) four coplanar, cocircular centres in the upper half: a singular tet solve; every slab that loads it
    # reports the same solve under the same global key
    c_deg, r_deg = c.copy(), r.copy()
    mid = np.argsort(c[:, 2])[12_000:12_004]
    base = c[mid[0]]
    c_deg[mid] = base + np.array([[0, 0, 0], [1.6, 0, 0], [0, 1.6, 0], [1.6, 1.6, 0]])
    r_deg[mid] = 1.5
    cfg = ax.PipelineConfig(alpha=1.0)
    ref = oracle.compute(c_deg, r_deg, 1.0)
    assert ref.status == oracle.DEGENERATE
    with pytest.raises(ax.DegenerateSimplex) as whole:
        ax.compute_alpha_complex_arrays(c_deg, r_deg, cfg)
    assert tuple(whole.value.vertices) == tuple(ref.error_vertices)
    jobs = [sharding.ShardedJob(c_deg, r_deg, cfg, q, 5, eng) for q in range(5)]
    errs = [job.local(raise_errors=False)[1] for job in jobs]
    assert any(e is not None for e in errs)
    hit = sharding.pick_error(errs)
    assert tuple(hit[1].vertices) == tuple(ref.error_vertices)
    with pytest.raises(ax.DegenerateSimplex) as sharded:
        eng.raise_slab_error(hit[1], cfg)
    assert str(sharded.value) == str(whole.value) and sharded.value.vertices == whole.value.vertices


def test_device_merge_rows_matches_numpy():
    import torch

    eng = ax.default_engine()
    rng = np.random.default_rng(5)
    for k in (1, 2, 3, 4):
        rows = np.sort(rng.integers(0, 500, size=(20_000, k)), axis=1)
        got = eng.merge_rows(torch.as_tensor(rows, device="cuda"), k, 500).cpu().numpy()
        want = np.unique(rows, axis=0)
        assert np.array_equal(got.reshape(-1, k), want)
    assert eng.merge_rows(torch.empty((0, 3), dtype=torch.int64, device="cuda"), 3, 10).shape[0] == 0
    # one index range of a sharded run: first indices in [200, 350)
    rows = np.sort(rng.integers(200, 500, size=(5_000, 3)), axis=1)
    rows = rows[rows[:, 0] < 350]
    got = eng.merge_rows(torch.as_tensor(rows, device="cuda"), 3, 350, index_lo=200).cpu().numpy()
    assert np.array_equal(got, np.unique(rows, axis=0))
    with pytest.raises(ax.AlphaxError):
        eng.merge_rows(torch.as_tensor(rows, device="cuda"), 3, 340, index_lo=200)


def test_standalone_stage_api_against_reference_golden(gold_small):
    """build_grid / potential_* / prune with the reference's names and result types."""
    for name in ("g1_200_a14", "tetra_a05", "profile0_s0_a1.2", "near_regular_a15"):
        rec = gold_small[name]
        m = rec["meta"]
        balls = [ax.Ball(tuple(c), float(r), i) for i, (c, r) in enumerate(zip(rec["centers"], rec["radii"]))]
        cfg = ax.PipelineConfig(alpha=m["alpha"], tolerance=ax.TolerancePolicy(m["eps_abs"], m["eps_singular"]))
        grid = ax.build_grid(balls, m["alpha"])
        st, g = oracle.grid_build(rec["centers"], rec["radii"], m["alpha"])
        assert grid.dims == g.dims and grid.cell_side == g.side and np.array_equal(grid.order, g.order)
        assert grid.range_offsets[-1] == len(balls) and (np.diff(grid.occupied_keys) > 0).all()
        edges = ax.potential_edges(grid, balls, cfg)
        tris = ax.potential_triangles(edges, grid, balls, cfg)
        tets = ax.potential_tets(tris, grid, balls, cfg)
        for d, lv in ((1, edges), (2, tris), (3, tets)):
            pm = m["potentials"][f"p{d}"]
            assert len(lv) == pm["count"]
            assert digest_arrays(lv.simplices) == pm["sha256_rows"]                    # rows as the reference lists them
            assert digest_values(lv.centers, lv.sizes) == pm["sha256_values"]          # cached fp64 ortho data, bitwise
            if m["potentials_stored"]:
                rows, cen, siz = rec[f"p{d}"]
                assert np.array_equal(lv.simplices, rows.reshape(lv.simplices.shape))
        k = ax.prune(ax.PotentialSets(edges=edges, triangles=tris, tets=tets, alpha=m["alpha"]), grid, balls, cfg)
        assert list(k.counts()) == m["counts"]
        assert hashlib.sha256(ax.write_complex(k).encode()).hexdigest() == m["sha256_complex"]
        assert ax.read_complex(ax.write_complex(k)) == k


def test_sparse_grid_mode(monkeypatch):
    """Widely spread inputs (the dense cell table would need > 2^31 cells) go through the sorted-key
    grid; forcing that mode on ordinary inputs must not change a bit either."""
    # two globules 2e6 A apart plus a stray ball: ~1e18 cells
    c1, r1 = synth.random_globule(400, 3, 1.0, (1.2, 1.9), 1 / 12)
    c2, r2 = synth.random_globule(300, 4, 1.0, (1.2, 1.9), 1 / 12)
    c = np.concatenate([c1, c2 + np.array([2.0e6, -1.5e6, 1.0e6]), np.array([[5.0e5, 5.0e5, 5.0e5]])])
    r = np.concatenate([r1, r2, [1.5]])
    perm = np.random.default_rng(1).permutation(len(r))
    c, r = np.ascontiguousarray(c[perm]), r[perm]
    for alpha in (0.0, 1.4):
        ref = oracle.compute(c, r, alpha, keep_potentials=True)
        assert ref.status == oracle.OK
        k = ax.compute_alpha_complex_arrays(c, r, ax.PipelineConfig(alpha=alpha))
        assert_same_complex(k, ref, f"sparse a={alpha}")
    grid = ax.build_grid([ax.Ball(tuple(p), float(q), i) for i, (p, q) in enumerate(zip(c, r))], 0.0)
    st, g = oracle.grid_build(c, r, 0.0)
    assert grid.dims == g.dims and np.array_equal(grid.order, g.order) and np.array_equal(grid.ball_cells, g.cells)
    # ordinary inputs, sparse mode forced
    monkeypatch.setenv("AXB_FORCE_SPARSE", "1")
    for (cc, rr), alpha, eps in ((synth.jittered_lattice(30_000, 6), 1.4, 1e-300),
                                 (synth.adversarial_density(20_000, 1, shuffle=True), 0.0, 1e-300),
                                 (synth.random_globule(160, 9, 0.35, (0.4, 1.6), 0.9), 1.0, 1e-300)):
        ref = oracle.compute(cc, rr, alpha, eps_singular=eps, threads=os.cpu_count(), chunk=2000)
        k = ax.compute_alpha_complex_arrays(cc, rr, ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps)))
        assert_same_complex(k, ref, "forced sparse")
    dup = np.array([[0, 0, 0], [1e7, 1, 1], [0, 0, 0.0]])
    with pytest.raises(ax.DuplicateCenter, match="balls 0 and 2 share"):
        ax.compute_alpha_complex_arrays(dup, np.array([1, 1, 1.5]), ax.PipelineConfig(alpha=0.0))


def test_compact_wire_formats_of_the_host_path(monkeypatch):
    """AXB_WIRE=3: edges / triangles cross PCIe without their owner column and are rebuilt by the host
    threads from the per-owner offsets; the int64 arrays must be identical to the default format."""
    eng = ax.default_engine()
    c, r = synth.jittered_lattice(120_000, 5)
    cfg = ax.PipelineConfig(alpha=0.7)
    plain = eng.compute_host(c, r, cfg)
    for mode in ("1", "2", "3"):
        monkeypatch.setenv("AXB_WIRE", mode)
        compact = eng.compute_host(c, r, cfg)
        for a, b in zip(plain, compact):
            assert a.dtype == np.int64 and np.array_equal(a, b), f"AXB_WIRE={mode}"
    monkeypatch.delenv("AXB_WIRE")
    # the default is the 24-bit format (ball indices < 2^24): three bytes per value, planes of low halves and high
    # bytes per D2H chunk; AXB_WIRE24=0 sends int32.  Small chunks make the lists span many (and ragged) chunks.
    two_call = eng.compute_host(c, r, cfg, pipelined=False)
    for chunk in ("", "16384", "50000"):
        if chunk:
            monkeypatch.setenv("AXB_D2H_CHUNK", chunk)
        for w24 in ("1", "0"):
            monkeypatch.setenv("AXB_WIRE24", w24)
            got = eng.compute_host(c, r, cfg)
            wire = int(eng.lib.axb_last_d2h_bytes(eng.handle))
            values = sum(int(a.size) for a in got[1:])
            assert wire == values * (3 if w24 == "1" else 4), (w24, chunk)
            for a, b in zip(two_call, got):
                assert a.dtype == np.int64 and np.array_equal(a, b), f"AXB_WIRE24={w24} chunk={chunk}"
    monkeypatch.delenv("AXB_WIRE24")
    monkeypatch.setenv("AXB_D2H_CHUNK", str(1 << 19))
    # vertices dropped by the general vertex step (not every vertex kept): the plain int32 path for dimension 0
    rng = np.random.default_rng(3)
    c2 = rng.uniform(0, 30, size=(3000, 3))
    r2 = rng.uniform(0.1, 2.5, size=3000)
    k = ax.compute_alpha_complex_arrays(c2, r2, ax.PipelineConfig(alpha=0.0, tolerance=ax.TolerancePolicy(1e-9, 1e-300)))
    ref = oracle.compute(c2, r2, 0.0, eps_singular=1e-300, threads=os.cpu_count(), chunk=64)
    assert ref.status == oracle.OK and k.vertices.shape[0] < 3000
    assert_same_complex(k, ref, "engulfed vertices")


def test_pipelined_host_path_equals_two_call_path():
    eng = ax.default_engine()
    cases = [(synth.jittered_lattice(120_000, 3), 0.0, 1e-300),
             (synth.jittered_lattice(40_000, 3), 1.4, 1e-300),
             (synth.random_globule(160, 9, 0.35, (0.4, 1.6), 0.9), 1.0, 1e-300),
             ((np.array([[0.0, 0, 0], [10, 0, 0]]), np.array([2.0, 0.5])), -1.0, 1e-12),
             ((np.array([[1.0, 2, 3]]), np.array([1.0])), 0.0, 1e-12)]
    for (c, r), alpha, eps in cases:
        cfg = ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps))
        a = eng.compute_host(c, r, cfg, pipelined=True)
        b = eng.compute_host(c, r, cfg, pipelined=False)
        for x, y in zip(a, b):
            assert x.dtype == np.int64 and np.array_equal(x, y)
