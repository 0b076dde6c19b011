#!/usr/bin/env python
"""Does overlapping several host-path calls on ONE GPU pay?  k engines (own context, stream, arena, staging
area), one host thread each, work through a list of alpha values; compared with one engine doing them in turn.

    python tools/gpu_sweep_probe.py [n_atoms] [engines] [repeats]
"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import Engine, PipelineConfig, TolerancePolicy, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
c, r = synth.jittered_lattice(n, 0)
hc, hr = torch.as_tensor(c).pin_memory().numpy(), torch.as_tensor(r).pin_memory().numpy()
tol = TolerancePolicy(1e-9, 1e-300)
alphas = [0.0, 1.4] * (reps // 2)
cfgs = [PipelineConfig(alpha=a, tolerance=tol) for a in alphas]


def serial(eng):
    t0 = time.perf_counter()
    for cfg in cfgs:
        eng.compute_host(hc, hr, cfg)
    return time.perf_counter() - t0


def overlapped(engs, streams):
    def work(i):
        with torch.cuda.stream(streams[i]):
            for j in range(i, len(cfgs), len(engs)):
                engs[i].compute_host(hc, hr, cfgs[j])
    th = [threading.Thread(target=work, args=(i,)) for i in range(len(engs))]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    return time.perf_counter() - t0


engs = [Engine(0) for _ in range(k)]
streams = [torch.cuda.Stream() for _ in range(k)]
for _ in range(2):
    serial(engs[0])
    overlapped(engs, streams)
ts = min(serial(engs[0]) for _ in range(3))
to = min(overlapped(engs, streams) for _ in range(3))
print(f"n={n} alphas={len(cfgs)} widen_threads={os.environ.get('AXB_WIDEN_THREADS', 'default')}: "
      f"one engine {ts * 1e3 / len(cfgs):.2f} ms per alpha, {k} engines overlapped {to * 1e3 / len(cfgs):.2f} ms per alpha")
