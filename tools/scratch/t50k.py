import sys, time, json
sys.path.insert(0, "/root/repo")
from dataclasses import replace
import numpy as np, torch
import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import synth
eng = ax.default_engine()
for n in (1000, 50_000):
    c, r = synth.jittered_lattice(n, 0)
    dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
    for eps in (1e-12, 1e-300):
        for a in (0.0, 0.6, 1.4):
            cfg = ax.PipelineConfig(alpha=a, tolerance=ax.TolerancePolicy(1e-9, eps))
            try:
                eng.compute_device(dc, dr, cfg)
            except Exception as e:
                print(n, eps, a, "raises", type(e).__name__); continue
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for _ in range(20): eng.compute_device(dc, dr, cfg)
            torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
            print(n, eps, a, f"{dt*1e3:.3f} ms", {k: round(v, 3) for k, v in eng.last_stage_ms.items()})
# sweep phases at 1M
c, r = synth.jittered_lattice(1_000_000, 0)
dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
cfg = ax.PipelineConfig(alpha=1.4, tolerance=ax.TolerancePolicy(1e-9, 1e-300))
import ctypes as C
def t(label, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    print(label, f"{(time.perf_counter()-t0)*1e3:.3f} ms"); return out
for rep in range(2):
    t("grid", lambda: eng.stage_grid(dc, dr, cfg))
    t("potential", lambda: eng.stage_potential())
    t("prepare", lambda: eng._stage_call(eng.lib.axb_sweep_prepare))
    for a in (0.0, 1.4):
        t(f"prune {a}", lambda: eng._stage_call(eng.lib.axb_sweep_prune, C.c_double(a)))
        cnt = t("canon", lambda: eng.stage_canonicalize())
        t("export", lambda: eng.stage_export(cnt))
