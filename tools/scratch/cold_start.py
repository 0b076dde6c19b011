#!/usr/bin/env python
"""First calls of a fresh process: wall time of call 1, 2, 3 ... of the device-resident and the host entry point."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
c, r = synth.jittered_lattice(n, 0)
cfg = ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
torch.cuda.init()
torch.zeros(1, device="cuda")
t0 = time.perf_counter()
eng = ax.default_engine()
print(f"engine created in {(time.perf_counter() - t0) * 1e3:.1f} ms")
dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs = eng.compute_device(dc, dr, cfg)
    torch.cuda.synchronize()
    print(f"compute_device call {i + 1}: {(time.perf_counter() - t0) * 1e3:.2f} ms, launches so far {eng.kernel_launches}")
for i in range(4):
    t0 = time.perf_counter()
    k = ax.compute_alpha_complex_arrays(c, r, cfg)
    print(f"compute_alpha_complex_arrays call {i + 1}: {(time.perf_counter() - t0) * 1e3:.2f} ms, launches so far {eng.kernel_launches}")
