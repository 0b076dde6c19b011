#!/usr/bin/env python
"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / initcheck):

    compute-sanitizer --tool memcheck python tools/gpu_sanitize.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import sharding, synth  # noqa: E402


def check(name, c, r, alpha, eps=1e-300):
    cfg = ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps))
    k = ax.compute_alpha_complex_arrays(c, r, cfg)
    ref = oracle.compute(c, r, alpha, eps_singular=eps)
    ok = all(np.array_equal(a, b) for a, b in zip((k.vertices, k.edges, k.triangles, k.tets),
                                                  (ref.vertices, ref.edges, ref.triangles, ref.tets)))
    print(name, k.counts(), "bit-exact" if ok else "MISMATCH", flush=True)
    return ok


def main():
    ok = True
    ok &= check("g2 3000 a=0", *synth.jittered_lattice(3000, 1), 0.0)
    ok &= check("g2 3000 a=1.4", *synth.jittered_lattice(3000, 1), 1.4)
    ok &= check("dense blob (W=4 path)", *synth.random_globule(160, 9, 0.35, (0.4, 1.6), 0.9), 1.0)
    ok &= check("adversarial 3000", *synth.adversarial_density(3000, 2), 0.0)
    os.environ["AXB_FORCE_SPARSE"] = "1"
    ok &= check("g2 2000 a=0.7 sparse grid", *synth.jittered_lattice(2000, 3), 0.7)
    del os.environ["AXB_FORCE_SPARSE"]
    # hundreds of partners per ball: k_edges_heavy (two-sweep lists), k_tri_tet_heavy (bit matrices in global scratch)
    rng = np.random.default_rng(5)
    n, rho = 520, 50.0
    th = np.linspace(0.0, 2.9 / rho, n)
    arc = np.stack([rho * np.cos(th), rho * np.sin(th), rng.uniform(-3e-3, 3e-3, size=n)], axis=1)[rng.permutation(n)]
    ok &= check("520 balls on an arc (up to ~500 partners)", arc, rng.uniform(1.45, 1.55, size=n), 0.0)
    # stage API on caller-edited levels (import kernels, tets from triangles, AC2 mask) and the alpha sweep
    c, r = synth.jittered_lattice(1500, 7)
    balls = [ax.Ball(tuple(p), float(q), i) for i, (p, q) in enumerate(zip(c, r))]
    cfg = ax.PipelineConfig(alpha=0.8, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
    grid = ax.build_grid(balls, 0.8)
    e = ax.potential_edges(grid, balls, cfg)
    thin = ax.PotentialLevel(simplices=e.simplices[::2], centers=e.centers[::2], sizes=e.sizes[::2])
    t = ax.potential_triangles(thin, grid, balls, cfg)
    q = ax.potential_tets(ax.PotentialLevel(simplices=t.simplices[1::2], centers=t.centers[1::2], sizes=t.sizes[1::2]), grid, balls, cfg)
    m = ax.ac2_mask(t, grid, balls, cfg)
    t_full = ax.potential_triangles(e, grid, balls, cfg)
    q_full = ax.potential_tets(t_full, grid, balls, cfg)
    k = ax.prune(ax.PotentialSets(edges=e, triangles=t_full, tets=q_full, alpha=0.8), grid, balls, cfg)
    ref = oracle.compute(c, r, 0.8, eps_singular=1e-300)
    same_k = all(np.array_equal(a, b) for a, b in zip((k.vertices, k.edges, k.triangles, k.tets), (ref.vertices, ref.edges, ref.triangles, ref.tets)))
    print("stage API (edited + complete levels)", len(t), len(q), int(m.sum()), "bit-exact" if same_k else "MISMATCH", flush=True)
    ok &= same_k
    sweep = ax.compute_alpha_sweep(c, r, [0.0, 0.8, -0.3], cfg)
    for a, ks in zip([0.0, 0.8, -0.3], sweep):
        ref = oracle.compute(c, r, a, eps_singular=1e-300)
        good = all(np.array_equal(x, y) for x, y in zip((ks.vertices, ks.edges, ks.triangles, ks.tets), (ref.vertices, ref.edges, ref.triangles, ref.tets)))
        print(f"sweep alpha={a}", ks.counts(), "bit-exact" if good else "MISMATCH", flush=True)
        ok &= good
    # the device path on remembered list lengths: same shape, denser / sparser point sets (held, redone, held)
    import torch

    eng = ax.default_engine()
    c, r = synth.jittered_lattice(6000, 14)
    r = r.copy()
    r[0] = 1.9
    mid = 0.5 * (c.min(axis=0) + c.max(axis=0))
    keep = np.unique(np.concatenate([c.argmin(axis=0), c.argmax(axis=0)]))
    cfg = ax.PipelineConfig(alpha=0.3, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
    for scale in (1.0, 1.0, 0.8, 0.8, 1.15):
        v = mid + (c - mid) * scale
        v[keep] = c[keep]
        v = np.ascontiguousarray(v)
        want = eng.compute_host(v, r, cfg)
        got = [t.cpu().numpy() for t in eng.compute_device(torch.as_tensor(v, device="cuda"), torch.as_tensor(r, device="cuda"), cfg)]
        good = all(np.array_equal(a, b) for a, b in zip(want, got))
        print(f"remembered sizes, scale {scale}", [g.shape[0] for g in got], "bit-exact" if good else "MISMATCH", flush=True)
        ok &= good
    c, r = synth.jittered_lattice(4000, 5)
    cfg = ax.PipelineConfig(alpha=0.5)
    single = eng.compute_host(c, r, cfg)
    merged, _ = sharding.compute_sharded_single_gpu(c, r, cfg, 3, eng)
    same = all(np.array_equal(m.cpu().numpy(), s) for m, s in zip(merged, single))
    print("3 slabs + device merge", "bit-exact" if same else "MISMATCH", flush=True)
    sys.exit(0 if (ok and same) else 1)


if __name__ == "__main__":
    main()
