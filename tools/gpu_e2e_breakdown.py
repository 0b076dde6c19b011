#!/usr/bin/env python
"""Where the end-to-end time of the host API goes (1M atoms, alpha 0, pinned inputs)."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import _native as N, synth  # noqa: E402


def main():
    c, r = synth.jittered_lattice(1_000_000, 0)
    hc, hr = torch.as_tensor(c).pin_memory().numpy(), torch.as_tensor(r).pin_memory().numpy()
    cfg = ax.PipelineConfig(alpha=0.0)
    eng = ax.default_engine()
    for mode in (True, False):
        for _ in range(3):
            eng.compute_host(hc, hr, cfg, pipelined=mode)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            out = eng.compute_host(hc, hr, cfg, pipelined=mode)
            del out
        print(f"compute_host pipelined={mode}: {(time.perf_counter() - t0) * 100:.3f} ms/call")
    # pageable inputs (a plain numpy array): staged through pinned memory by the host threads
    for _ in range(3):
        eng.compute_host(c, r, cfg)
    t0 = time.perf_counter()
    for _ in range(10):
        out = eng.compute_host(c, r, cfg)
        del out
    print(f"compute_host pageable inputs: {(time.perf_counter() - t0) * 100:.3f} ms/call")
    # raw phases of the pipelined path
    lib, h = eng.lib, eng.handle
    prm = eng._params(cfg)
    cap, counts = (C.c_int64 * 4)(), (C.c_int64 * 4)()
    tb = ta = tf = 0.0
    for _ in range(10):
        t0 = time.perf_counter()
        assert lib.axb_compute_host_begin(h, len(r), hc.ctypes.data, hr.ctypes.data, C.byref(prm), cap) == 0
        t1 = time.perf_counter()
        outs = [torch.empty((int(cap[d]),) if d == 0 else (int(cap[d]), d + 1), dtype=torch.int64, pin_memory=True).numpy()
                for d in range(4)]
        t2 = time.perf_counter()
        assert lib.axb_compute_host_finish(h, *(o.ctypes.data for o in outs), counts) == 0
        t3 = time.perf_counter()
        tb += t1 - t0; ta += t2 - t1; tf += t3 - t2
        del outs
    print(f"begin {tb * 100:.3f} ms, pinned alloc {ta * 100:.3f} ms, finish {tf * 100:.3f} ms  caps {list(cap)} counts {list(counts)}")
    tb = ta = tf = 0.0
    for _ in range(10):
        t0 = time.perf_counter()
        assert lib.axb_compute_host_begin(h, len(r), c.ctypes.data, r.ctypes.data, C.byref(prm), cap) == 0
        t1 = time.perf_counter()
        outs = [torch.empty((int(cap[d]),) if d == 0 else (int(cap[d]), d + 1), dtype=torch.int64, pin_memory=True).numpy()
                for d in range(4)]
        t2 = time.perf_counter()
        assert lib.axb_compute_host_finish(h, *(o.ctypes.data for o in outs), counts) == 0
        t3 = time.perf_counter()
        tb += t1 - t0; ta += t2 - t1; tf += t3 - t2
        del outs
    print(f"pageable inputs: begin {tb * 100:.3f} ms, pinned alloc {ta * 100:.3f} ms, finish {tf * 100:.3f} ms")
    # pure copies for reference
    d = torch.empty(181658136 // 8, dtype=torch.int64, device="cuda")
    hp = torch.empty(181658136 // 8, dtype=torch.int64, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        hp.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
    print(f"pure D2H of 182 MB: {(time.perf_counter() - t0) * 100:.3f} ms")
    di = torch.empty(4_000_000, dtype=torch.float64, device="cuda")
    hi = torch.empty(4_000_000, dtype=torch.float64, pin_memory=True)
    t0 = time.perf_counter()
    for _ in range(10):
        di.copy_(hi, non_blocking=True)
        torch.cuda.synchronize()
    print(f"pure H2D of 32 MB: {(time.perf_counter() - t0) * 100:.3f} ms")


if __name__ == "__main__":
    main()
