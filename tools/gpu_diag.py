#!/usr/bin/env python
"""Stage-by-stage comparison of the CUDA path with the CPU oracle on a GPU box.

    python tools/gpu_diag.py [--big]

Prints, per input, which stage first disagrees (grid order, potential edges /
triangles / tets incl. cached ortho data, final complex) with a few differing
rows.  A debugging aid; the pass/fail record is tests/test_gpu_*.py.
"""
import json
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1908_05944_b200 import Engine, PipelineConfig, TolerancePolicy, synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def lexsort_rows(rows):
    if rows.shape[0] == 0:
        return np.empty(0, dtype=np.int64)
    return np.lexsort(tuple(rows[:, c] for c in range(rows.shape[1] - 1, -1, -1)))


def show_diff(name, got, want, limit=5):
    gs = {tuple(r) for r in got.reshape(got.shape[0], -1).tolist()}
    ws = {tuple(r) for r in want.reshape(want.shape[0], -1).tolist()}
    extra = sorted(gs - ws)[:limit]
    missing = sorted(ws - gs)[:limit]
    print(f"    {name}: got {got.shape[0]} want {want.shape[0]}; extra {len(gs - ws)} e.g. {extra}; "
          f"missing {len(ws - gs)} e.g. {missing}; dup rows in got: {got.shape[0] - len(gs)}")


def run_case(eng, name, c, r, alpha, eps_abs=1e-9, eps_sing=1e-12, bio=False):
    cfg = PipelineConfig(alpha=alpha, biomolecule_mode=bio, tolerance=TolerancePolicy(eps_abs, eps_sing))
    ref = oracle.compute(c, r, alpha, eps_abs=eps_abs, eps_singular=eps_sing, biomolecule=bio,
                         keep_potentials=True, threads=os.cpu_count(), chunk=max(1, len(r) // 64))
    ok = True
    t0 = time.time()
    try:
        dc = torch.as_tensor(c, device="cuda")
        dr = torch.as_tensor(r, device="cuda")
        info = eng.stage_grid(dc, dr, cfg)
        st, g = oracle.grid_build(c, r, alpha)
        order, rank, cells = (t.cpu().numpy() for t in eng.stage_grid_export())
        if not (info["dims"] == g.dims and info["cell_side"] == g.side and np.array_equal(info["origin"], g.origin)):
            print(f"  [{name}] GRID GEOMETRY differs: {info} vs side={g.side} dims={g.dims} origin={g.origin}")
            ok = False
        for nm, a, b in (("order", order, g.order), ("rank", rank, g.rank), ("cells", cells, g.cells)):
            if not np.array_equal(a, b):
                bad = np.flatnonzero(a != b)
                print(f"  [{name}] GRID {nm} differs at {bad.size} places, first {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}")
                ok = False
        pc = eng.stage_potential()
        for dim in (1, 2, 3):
            rows, cen, siz = (t.cpu().numpy() for t in eng.stage_potential_export(dim))
            perm = lexsort_rows(rows)
            rows, cen, siz = rows[perm], cen[perm], siz[perm]
            wrows, wcen, wsiz = ref.potentials[dim]
            if not np.array_equal(rows, wrows):
                print(f"  [{name}] POTENTIAL dim {dim} rows differ")
                show_diff(f"p{dim}", rows, wrows)
                ok = False
            elif not (np.array_equal(cen.view(np.uint64), wcen.view(np.uint64)) and
                      np.array_equal(siz.view(np.uint64), wsiz.view(np.uint64))):
                bad = np.flatnonzero((siz != wsiz) | (cen != wcen).any(axis=1))
                print(f"  [{name}] POTENTIAL dim {dim}: rows equal, ortho data differs at {bad.size} rows; "
                      f"max |dsize| {np.abs(siz - wsiz).max():.3e}")
                ok = False
        eng.stage_prune()
        counts = eng.stage_canonicalize()
        outs = [t.cpu().numpy() for t in eng.stage_export(counts)]
        for d, (got, want) in enumerate(zip(outs, (ref.vertices, ref.edges, ref.triangles, ref.tets))):
            if not np.array_equal(got, want):
                print(f"  [{name}] COMPLEX dim {d} differs")
                show_diff(f"k{d}", got.reshape(got.shape[0], -1), want.reshape(want.shape[0], -1))
                if got.shape == want.shape:
                    print(f"    same set, different order: {sorted(map(tuple, got.reshape(got.shape[0], -1).tolist())) == list(map(tuple, want.reshape(want.shape[0], -1).tolist()))}")
                ok = False
        ms = eng.last_stage_ms
        print(f"  [{name}] n={len(r)} alpha={alpha} {'OK ' if ok else 'FAIL'} potentials={pc} complex={counts} "
              f"oracle={ref.counts()} wall={time.time() - t0:.3f}s stage_ms=" +
              ",".join(f"{k}:{v:.3f}" for k, v in ms.items()))
    except Exception as e:  # noqa: BLE001
        ok = False
        print(f"  [{name}] EXCEPTION {type(e).__name__}: {e}")
        traceback.print_exc(limit=3)
    return ok


def main():
    big = "--big" in sys.argv
    print("device:", torch.cuda.get_device_name(0))
    eng = Engine(0)
    eng.stage_timing = True          # this tool reads eng.last_stage_ms
    allok = True
    # 1. predicate arithmetic
    d = np.load(os.path.join(GOLD, "ortho_vectors.npz"))
    for k in (1, 2, 3, 4):
        cen, siz, sg = eng.ortho_batch(d[f"k{k}_points"], d[f"k{k}_r2"], 1e-12)
        wsg = d[f"k{k}_eps1e-12_singular"]
        good = ~wsg
        same = (np.array_equal(sg, wsg) and
                np.array_equal(cen[good].view(np.uint64), d[f"k{k}_eps1e-12_centers"][good].view(np.uint64)) and
                np.array_equal(siz[good].view(np.uint64), d[f"k{k}_eps1e-12_sizes"][good].view(np.uint64)))
        print(f"ortho k={k}: {'bitwise OK' if same else 'MISMATCH'}"
              + ("" if same else f" max|dsize|={np.abs(siz[good] - d[f'k{k}_eps1e-12_sizes'][good]).max():.3e} singular_equal={np.array_equal(sg, wsg)}"))
        allok &= same
    # 2. golden small cases, stage by stage
    data = np.load(os.path.join(GOLD, "complex_small.npz"))
    index = json.load(open(os.path.join(GOLD, "complex_small.json")))
    for name, m in index.items():
        allok &= run_case(eng, name, data[name + "__centers"], data[name + "__radii"], m["alpha"], m["eps_abs"],
                          m["eps_singular"], m["biomolecule"])
    # 3. generator configs
    for n, alpha in ((1000, 0.0), (1000, 1.4)):
        c, r = synth.random_globule(n, 0, 1.0, (1.2, 1.9), 1 / 12)
        allok &= run_case(eng, f"config1_a{alpha}", c, r, alpha)
    for n, alpha in ((50_000, 0.0), (50_000, 1.4)) + (((200_000, 0.0), (1_000_000, 0.0)) if big else ()):
        c, r = synth.jittered_lattice(n, 0)
        allok &= run_case(eng, f"g2_{n}_a{alpha}", c, r, alpha, eps_sing=1e-12 if n < 1_000_000 else 1e-12)
    c, r = synth.adversarial_density(100_000 if big else 20_000, 0)
    allok &= run_case(eng, "adversarial", c, r, 0.0, eps_sing=1e-300)
    print("ALL OK" if allok else "SOME FAILED")
    return 0 if allok else 1


if __name__ == "__main__":
    sys.exit(main())
