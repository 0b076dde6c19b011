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
    c, r = synth.jittered_lattice(4000, 5)
    cfg = ax.PipelineConfig(alpha=0.5)
    eng = ax.default_engine()
    single = eng.compute_host(c, r, cfg)
    merged, _ = sharding.compute_sharded_single_gpu(c, r, cfg, 3, eng)
    same = all(np.array_equal(m.cpu().numpy(), s) for m, s in zip(merged, single))
    print("3 slabs + device merge", "bit-exact" if same else "MISMATCH", flush=True)
    sys.exit(0 if (ok and same) else 1)


if __name__ == "__main__":
    main()
