#!/usr/bin/env python
"""Stage-time table of the CUDA path for a few workloads (device-resident, CUDA events inside the
library).  A development aid for A/B comparisons; bench.py is the record.

    python tools/gpu_perf.py [reps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_05944_b200 import Engine, PipelineConfig, TolerancePolicy, synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    eng = Engine(0)
    eng.stage_timing = True          # this tool reads eng.last_stage_ms
    tol = TolerancePolicy(1e-9, 1e-300)
    work = [("g2_1M_a0", synth.jittered_lattice(1_000_000, 0), 0.0),
            ("g2_1M_a1.4", synth.jittered_lattice(1_000_000, 0), 1.4),
            ("adv_1M_a0", synth.adversarial_density(1_000_000, 0), 0.0),
            ("g2_50k_a0", synth.jittered_lattice(50_000, 0), 0.0)]
    keys = None
    for name, (c, r), alpha in work:
        cfg = PipelineConfig(alpha=alpha, tolerance=tol)
        dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
        for _ in range(2):
            outs = eng.compute_device(dc, dr, cfg)
        acc = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            outs = eng.compute_device(dc, dr, cfg)
            for k, v in eng.last_stage_ms.items():
                acc[k] = acc.get(k, 0.0) + v / reps
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps * 1e3
        if keys is None:
            keys = list(acc)
            print("workload        counts                                 wall_ms  sum_ms  " + " ".join(f"{k[:9]:>9s}" for k in keys))
        counts = tuple(int(o.shape[0]) for o in outs)
        print(f"{name:14s} {str(counts):40s} {wall:7.3f} {sum(acc.values()):7.3f}  " + " ".join(f"{acc[k]:9.3f}" for k in keys))


if __name__ == "__main__":
    main()
