#!/usr/bin/env python
"""Fixed cost of one call on small inputs (a typical protein has 1k-50k atoms): public API, engine call, the
two C-ABI phases, and the device-resident path.

    python tools/gpu_small_latency.py [n ...]
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import synth  # noqa: E402


def timeit(f, reps):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [1000, 10_000, 50_000]
    eng = ax.default_engine()
    lib, h = eng.lib, eng.handle
    for n in sizes:
        c, r = synth.jittered_lattice(n, 0)
        cfg = ax.PipelineConfig(alpha=0.0)
        dc, dr = torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda")
        prm = eng._params(cfg)
        cap, counts = (C.c_int64 * 4)(), (C.c_int64 * 4)()
        reps = 200
        t_api = timeit(lambda: ax.compute_alpha_complex_arrays(c, r, cfg), reps)
        t_host = timeit(lambda: eng.compute_host(c, r, cfg), reps)
        t_dev = timeit(lambda: eng.compute_device(dc, dr, cfg), reps)
        ph = [0.0, 0.0, 0.0]

        def phases():
            t0 = time.perf_counter()
            assert lib.axb_compute_host_begin(h, n, c.ctypes.data, r.ctypes.data, C.byref(prm), cap) == 0
            t1 = time.perf_counter()
            outs = [torch.empty((int(cap[d]),) if d == 0 else (int(cap[d]), d + 1), dtype=torch.int64, pin_memory=True).numpy()
                    for d in range(4)]
            t2 = time.perf_counter()
            assert lib.axb_compute_host_finish(h, *(o.ctypes.data for o in outs), counts) == 0
            t3 = time.perf_counter()
            ph[0] += t1 - t0; ph[1] += t2 - t1; ph[2] += t3 - t2

        timeit(phases, reps)
        k = 1e3 / (reps + 5)
        with eng.timing_stages():           # the latencies above are measured without stage events (the default)
            t_dev_timed = timeit(lambda: eng.compute_device(dc, dr, cfg), reps)
            stage = sum(eng.last_stage_ms.values())
        print(f"n={n}: public API {t_api:.3f} ms | engine host path {t_host:.3f} | begin {ph[0] * k:.3f} + pinned alloc "
              f"{ph[1] * k:.3f} + finish {ph[2] * k:.3f} | device-resident call {t_dev:.3f} ({t_dev_timed:.3f} with stage events, stage sum {stage:.3f})", flush=True)


if __name__ == "__main__":
    main()
