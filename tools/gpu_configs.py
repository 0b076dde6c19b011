#!/usr/bin/env python
"""The BASELINE.json configurations on one B200: wall time of the public host API call, device stage
sum, and bit-exactness against the CPU oracle (run on the box's host threads).

    python tools/gpu_configs.py [--with-10m]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import synth  # noqa: E402


def run(name, c, r, alpha, eps_sing, check=True):
    cfg = ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps_sing))
    eng = ax.default_engine()
    eng.stage_timing = True          # this tool reads eng.last_stage_ms
    ax.compute_alpha_complex_arrays(c, r, cfg)                       # warm-up (arena growth, pinned buffers)
    t0 = time.perf_counter()
    k = ax.compute_alpha_complex_arrays(c, r, cfg)
    wall = time.perf_counter() - t0
    dev = sum(eng.last_stage_ms.values())
    rec = dict(config=name, atoms=len(r), alpha=alpha, counts=list(k.counts()), e2e_ms=round(wall * 1e3, 2),
               device_stage_sum_ms=round(dev, 3), atoms_per_s_e2e=round(len(r) / wall), atoms_per_s_device=round(len(r) / dev * 1e3))
    if check:
        threads = os.cpu_count()
        t0 = time.perf_counter()
        ref = oracle.compute(c, r, alpha, eps_singular=eps_sing, threads=threads, chunk=max(1, len(r) // (8 * threads)))
        rec["cpu_oracle_s"] = round(time.perf_counter() - t0, 2)
        rec["cpu_threads"] = threads
        rec["bit_exact"] = bool(ref.status == oracle.OK and all(
            np.array_equal(a, b) for a, b in zip((k.vertices, k.edges, k.triangles, k.tets),
                                                 (ref.vertices, ref.edges, ref.triangles, ref.tets))))
    print(json.dumps(rec), flush=True)


def main():
    c, r = synth.random_globule(1000, 0, 1.0, (1.2, 1.9), 1 / 12)
    run("1: 1k globule a=0", c, r, 0.0, 1e-12)
    c, r = synth.jittered_lattice(50_000, 0)
    run("2: 50k a=0", c, r, 0.0, 1e-12)
    run("2: 50k a=1.4", c, r, 1.4, 1e-12)
    c, r = synth.jittered_lattice(1_000_000, 0)
    run("3: 1M a=0", c, r, 0.0, 1e-12)
    run("3: 1M a=1.4 (eps_singular 1e-300)", c, r, 1.4, 1e-300)
    c, r = synth.adversarial_density(1_000_000, 0)
    run("5: adversarial 1M a=0 (eps_singular 1e-300)", c, r, 0.0, 1e-300)
    if "--with-10m" in sys.argv:
        c, r = synth.jittered_lattice(10_000_000, 0)
        run("4: 10M a=0 on ONE gpu (eps_singular 1e-300)", c, r, 0.0, 1e-300, check="--check-10m" in sys.argv)


if __name__ == "__main__":
    main()
