import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1908_05944_b200 import Engine, PipelineConfig, TolerancePolicy, synth
eng = Engine(0)
out=[]
for n in (1000, 10000, 50000, 90000, 150000, 300000):
    c, r = synth.jittered_lattice(n, 0)
    dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
    cfg = PipelineConfig(alpha=0.0, tolerance=TolerancePolicy(1e-9, 1e-300))
    acc=0.0
    for i in range(13):
        eng.compute_device(dc, dr, cfg)
        if i>=3: acc += eng.last_stage_ms["potential_triangles"]/10
    out.append(f"n={n}: {acc*1000:.1f}us")
print("  ".join(out))
