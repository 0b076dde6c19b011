#!/usr/bin/env python
"""Large single-GPU runs against the CPU oracle: 10M atoms (24-bit wire, hundreds of D2H chunks per list) and
17M atoms (ball indices beyond 2^24: int32 wire).

    python tools/gpu_large_check.py [n ...]
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

for n in [int(a) for a in sys.argv[1:]] or [10_000_000, 17_000_000]:
    c, r = synth.jittered_lattice(n, 0)
    cfg = ax.PipelineConfig(alpha=0.0, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
    eng = ax.default_engine()
    eng.stage_timing = True          # this tool reads eng.last_stage_ms
    ax.compute_alpha_complex_arrays(c, r, cfg)
    t0 = time.perf_counter()
    k = ax.compute_alpha_complex_arrays(c, r, cfg)
    wall = time.perf_counter() - t0
    wire = int(eng.lib.axb_last_d2h_bytes(eng.handle))
    threads = os.cpu_count()
    t0 = time.perf_counter()
    ref = oracle.compute(c, r, 0.0, eps_singular=1e-300, threads=threads, chunk=max(1, n // (8 * threads)))
    cpu = time.perf_counter() - t0
    same = bool(ref.status == oracle.OK and all(np.array_equal(a, b) for a, b in zip(
        (k.vertices, k.edges, k.triangles, k.tets), (ref.vertices, ref.edges, ref.triangles, ref.tets))))
    values = int(k.edges.size + k.triangles.size + k.tets.size)
    print(json.dumps(dict(atoms=n, counts=list(k.counts()), e2e_ms=round(wall * 1e3, 2), wire_bytes=wire,
                          bytes_per_value=round(wire / values, 3), device_stage_sum_ms=round(sum(eng.last_stage_ms.values()), 3),
                          cpu_oracle_s=round(cpu, 1), cpu_threads=threads, bit_exact=same)), flush=True)
    del k, ref
