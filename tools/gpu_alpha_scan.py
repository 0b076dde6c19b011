#!/usr/bin/env python
"""Stage times of the potential triangle/tet kernel and of the tet pruning kernel over a range of alpha (1M atoms): where the light and the heavy
tile shape of k_tri_tet3 cross over (build with -DT3_HEAVY_PAIRS=0 / 100000 to force one of them).

    python tools/gpu_alpha_scan.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_05944_b200 import Engine, PipelineConfig, TolerancePolicy, synth  # noqa: E402

c, r = synth.jittered_lattice(1_000_000, 0)
dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
eng = Engine(0)
eng.stage_timing = True          # this tool reads eng.last_stage_ms
out = []
for alpha in (0.0, 0.2, 0.4, 0.6, 0.8, 1.0, 1.4):
    cfg = PipelineConfig(alpha=alpha, tolerance=TolerancePolicy(1e-9, 1e-300))
    acc = acc2 = 0.0
    for i in range(5):
        eng.compute_device(dc, dr, cfg)
        if i >= 2:
            acc += eng.last_stage_ms["potential_triangles"] / 3
            acc2 += eng.last_stage_ms["prune_tets"] / 3
    out.append(f"a={alpha}: {acc:.3f}/{acc2:.3f}")
print("  ".join(out))
