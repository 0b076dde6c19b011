#!/usr/bin/env python
"""Alpha sweep with re-use (csrc/sweep.cuh) against independent runs: device time per sweep on resident inputs.
    python tools/gpu_sweep_reuse.py [n] [alpha ...]"""
import json
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
alphas = [float(a) for a in sys.argv[2:]] or [0.0, 0.35, 0.7, 1.05, 1.4]
c, r = synth.jittered_lattice(n, 0)
eng = ax.default_engine()
cfg = ax.PipelineConfig(alpha=0.0, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")


def timed(fn, reps=8):
    out = None
    for _ in range(3):          # the caching allocator needs a few rounds before the result tensors stop costing cudaMalloc
        del out
        out = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        del out
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


t_sweep, sw = timed(lambda: eng.sweep_device(dc, dr, alphas, cfg))
t_alone, al = timed(lambda: [eng.compute_device(dc, dr, replace(cfg, alpha=a)) for a in alphas])
same = all(bool(torch.equal(x, y)) for s, a in zip(sw, al) for x, y in zip(s, a))
print(json.dumps({"n": n, "alphas": alphas, "sweep_ms": t_sweep, "independent_ms": t_alone, "identical": same,
                  "counts": [[int(x.shape[0]) for x in s] for s in sw]}))
