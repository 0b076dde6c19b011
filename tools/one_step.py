#!/usr/bin/env python
"""A few device-resident passes of one workload, for profilers (ncu -k regex:<kernel> -c 1 ...).

    python tools/one_step.py [n_atoms] [alpha] [passes]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_05944_b200 import Engine, PipelineConfig, TolerancePolicy, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
passes = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c, r = synth.jittered_lattice(n, 0)
eng = Engine(0)
eng.stage_timing = True          # this tool reads eng.last_stage_ms
cfg = PipelineConfig(alpha=alpha, tolerance=TolerancePolicy(1e-9, 1e-300))
dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
for _ in range(passes):
    outs = eng.compute_device(dc, dr, cfg)
torch.cuda.synchronize()
print([int(o.shape[0]) for o in outs], eng.last_stage_ms)
