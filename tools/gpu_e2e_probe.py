import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import synth
c,r=synth.jittered_lattice(1000000,0)
hc, hr = torch.as_tensor(c).pin_memory().numpy(), torch.as_tensor(r).pin_memory().numpy()
cfg=ax.PipelineConfig(alpha=0.0)
for i in range(4): ax.compute_alpha_complex_arrays(hc,hr,cfg)
best=1e9; tot=0
for i in range(20):
    t0=time.perf_counter(); ax.compute_alpha_complex_arrays(hc,hr,cfg); dt=time.perf_counter()-t0; best=min(best,dt); tot+=dt
print(os.environ.get("AXB_D2H_CHUNK","default"), os.environ.get("AXB_WIDEN_THREADS","default"), "mean %.3f ms best %.3f ms" % (tot/20*1e3, best*1e3))
