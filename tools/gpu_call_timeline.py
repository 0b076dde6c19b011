#!/usr/bin/env python
"""Timeline of ONE warm device-resident call (CUPTI through torch.profiler): every kernel / memset with its start
and duration, every CUDA runtime call on the host with its duration -- to see what a small input spends its time on.

    python tools/gpu_call_timeline.py [n] [alpha]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
c, r = synth.jittered_lattice(n, 0)
eng = ax.default_engine()
cfg = ax.PipelineConfig(alpha=alpha)
dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
for _ in range(20):
    eng.compute_device(dc, dr, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        out = eng.compute_device(dc, dr, cfg)
    torch.cuda.synchronize()
ev = sorted(prof.events(), key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
last_end = {}
for e in ev:
    dev = "GPU" if e.device_type == torch.autograd.DeviceType.CUDA else "cpu"
    name = e.name
    if dev == "cpu" and not name.startswith("cuda"):
        continue
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = s - last_end.get(dev, s)
    last_end[dev] = e.time_range.end - t0
    print(f"{dev} {s:9.1f} us  +{d:7.1f}  gap {gap:7.1f}  {name[:90]}")
