"""Pins the C oracle (oracle/) against the REAL reference's outputs.

Fixtures in tests/golden were produced by tools/make_golden.py importing the
reference package; every comparison here is exact (bitwise for floats).
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
from paper_1908_05944_b200 import synth

from conftest import GOLD
from helpers import canonical_text, digest_arrays, digest_values


def test_ortho_vectors_bitwise():
    d = np.load(os.path.join(GOLD, "ortho_vectors.npz"))
    for k in (1, 2, 3, 4):
        for eps in ("1e-12", "1e-300"):
            c, s, g = oracle.ortho_batch(d[f"k{k}_points"], d[f"k{k}_r2"], float(eps))
            ref_g = d[f"k{k}_eps{eps}_singular"]
            assert np.array_equal(g, ref_g)
            ok = ~ref_g   # rows of singular systems are documented as meaningless (geometry.py:127-128)
            assert np.array_equal(c[ok].view(np.uint64), d[f"k{k}_eps{eps}_centers"][ok].view(np.uint64))
            assert np.array_equal(s[ok].view(np.uint64), d[f"k{k}_eps{eps}_sizes"][ok].view(np.uint64))
        assert d[f"k{k}_eps1e-12_singular"].sum() > 0 or k < 3


def test_ortho_known_answers():
    # closed forms of the reference's T/test_geometry.py:29-69
    c, s, g = oracle.ortho_batch(np.array([[[0, 0, 0], [4, 0, 0.0]]]), np.array([[1.0, 1.0]]))
    assert np.allclose(c, [[2, 0, 0]]) and s[0] == pytest.approx(3.0) and not g[0]
    c, s, g = oracle.ortho_batch(np.array([[[0, 0, 0], [1, 0, 0.0]]]), np.array([[4.0, 0.25]]))
    assert c[0, 0] == pytest.approx(2.375) and s[0] == pytest.approx(1.640625)
    tri = np.array([[[0, 0, 0], [2, 0, 0], [1, np.sqrt(3.0), 0]]])
    c, s, g = oracle.ortho_batch(tri, np.ones((1, 3)))
    assert s[0] == pytest.approx(1.0 / 3.0, abs=1e-12)
    h = 2.0 * np.sqrt(6.0) / 3.0
    tet = np.array([[[0, 0, 0], [2, 0, 0], [1, np.sqrt(3.0), 0], [1, 1 / np.sqrt(3.0), h]]])
    c, s, g = oracle.ortho_batch(tet, np.ones((1, 4)))
    assert s[0] == pytest.approx(0.5, abs=1e-12)
    # collinear / coplanar / duplicate -> singular (T/test_geometry.py:115-135)
    assert oracle.ortho_batch(np.array([[[0, 0, 0], [1, 0, 0], [2, 0, 0.0]]]), np.ones((1, 3)))[2][0]
    assert oracle.ortho_batch(np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0.0]]]), np.ones((1, 4)))[2][0]
    assert oracle.ortho_batch(np.array([[[1, 1, 1], [1, 1, 1.0]]]), np.ones((1, 2)))[2][0]


def test_grid_vectors():
    d = np.load(os.path.join(GOLD, "grid_vectors.npz"))
    names = sorted({f.rsplit("_", 1)[0] for f in d.files if f.endswith("_order")})
    assert len(names) == 4
    for name in names:
        st, g = oracle.grid_build(d[name + "_centers"], d[name + "_radii"], float(d[name + "_alpha"]))
        assert st == oracle.OK
        assert g.side == float(d[name + "_side"])
        assert np.array_equal(g.origin, d[name + "_origin"])
        assert g.dims == tuple(int(v) for v in d[name + "_dims"])
        assert np.array_equal(g.order, d[name + "_order"])
        assert np.array_equal(g.rank, d[name + "_rank"])
        assert np.array_equal(g.cells, d[name + "_cells"])


def test_small_complexes_and_potentials(gold_small):
    assert len(gold_small) >= 40
    for name, rec in gold_small.items():
        m = rec["meta"]
        n = len(rec["radii"])
        for chunk, threads in ((None, 1), (7, 3)):
            o = oracle.compute(rec["centers"], rec["radii"], m["alpha"], eps_abs=m["eps_abs"],
                               eps_singular=m["eps_singular"], biomolecule=m["biomolecule"],
                               chunk=chunk, threads=threads, keep_potentials=True)
            assert o.status == oracle.OK, name
            assert list(o.counts()) == m["counts"], name
            for d, got in enumerate((o.vertices, o.edges, o.triangles, o.tets)):
                assert np.array_equal(got, rec[f"k{d}"].reshape(got.shape)), (name, d)
            text = canonical_text(o.vertices, o.edges, o.triangles, o.tets, n, m["alpha"])
            assert hashlib.sha256(text.encode()).hexdigest() == m["sha256_complex"], name
            for d in (1, 2, 3):
                rows, cen, siz = o.potentials[d]
                pm = m["potentials"][f"p{d}"]
                assert rows.shape[0] == pm["count"], (name, d)
                assert digest_arrays(rows) == pm["sha256_rows"], (name, d)
                assert digest_values(cen, siz) == pm["sha256_values"], (name, d)
                if m["potentials_stored"]:
                    assert np.array_equal(rows, rec[f"p{d}"][0].reshape(rows.shape))
                    assert np.array_equal(cen.view(np.uint64), rec[f"p{d}"][1].view(np.uint64).reshape(cen.shape))


def test_config1_golden(gold_config1):
    data, meta = gold_config1
    c, r = synth.random_globule(1000, 0, 1.0, (1.2, 1.9), 1 / 12)
    assert np.array_equal(c, data["centers"]) and np.array_equal(r, data["radii"])
    assert meta["a0"]["counts"] == [1000, 3705, 3268, 845]
    assert meta["a1.4"]["counts"] == [1000, 5336, 7008, 2697]
    assert meta["a0"]["sha256_complex"].startswith("00b61c8547390672")
    assert meta["a1.4"]["sha256_complex"].startswith("83fc6638225218e0")
    for tag, m in meta.items():
        o = oracle.compute(c, r, m["alpha"], biomolecule=m["biomolecule"], chunk=64, threads=2)
        assert list(o.counts()) == m["counts"]
        for d, got in enumerate((o.vertices, o.edges, o.triangles, o.tets)):
            assert np.array_equal(got, data[f"{tag}__k{d}"].reshape(got.shape))
        text = canonical_text(o.vertices, o.edges, o.triangles, o.tets, 1000, m["alpha"])
        assert hashlib.sha256(text.encode()).hexdigest() == m["sha256_complex"]


def test_error_cases(gold_errors):
    want_code = {"DegenerateSimplex": oracle.DEGENERATE, "DuplicateCenter": oracle.DUPLICATE,
                 "NonFiniteCoordinate": oracle.NONFINITE, "ValueError": oracle.BAD_SIDE, None: oracle.OK}
    for name, rec in gold_errors.items():
        o = oracle.compute(np.array(rec["centers"], dtype=np.float64), np.array(rec["radii"], dtype=np.float64),
                           rec["alpha"], eps_singular=rec["eps_singular"])
        assert o.status == want_code[rec["error"]], name
        if rec["error"] == "DegenerateSimplex":
            assert list(o.error_vertices) == rec["vertices"], name
        if rec["error"] == "DuplicateCenter":
            i, j = o.error_vertices
            assert rec["message"].startswith(f"balls {i} and {j} share"), name
    assert oracle.compute(np.empty((0, 3)), np.empty(0), 0.0).status == oracle.EMPTY
    bad = oracle.compute(np.array([[0, 0, 0], [np.nan, 0, 0]]), np.ones(2), 0.0)
    assert bad.status == oracle.NONFINITE and bad.error_vertices == (1,)
    bad = oracle.compute(np.array([[0, 0, 0], [1.0, 0, 0]]), np.array([1.0, np.inf]), 0.0)
    assert bad.status == oracle.NONFINITE and bad.error_vertices == (1,)


@pytest.mark.slow
def test_large_configs(gold_large):
    """50k / 200k-atom G2 configurations: counts and digest of the four arrays."""
    if not gold_large:
        pytest.skip("tests/golden/large_configs.json not generated")
    ran = 0
    for name, m in gold_large.items():
        if m["n"] > 200_000:
            continue      # the 1M cases are checked on the GPU box (tests/test_gpu_parity.py)
        c, r = synth.jittered_lattice(m["n"], m["seed"])
        o = oracle.compute(c, r, m["alpha"], eps_singular=m["eps_singular"], chunk=4000, threads=os.cpu_count())
        assert list(o.counts()) == m["counts"], name
        assert digest_arrays(o.vertices, o.edges, o.triangles, o.tets) == m["sha256_arrays"], name
        ran += 1
    assert ran >= 1
