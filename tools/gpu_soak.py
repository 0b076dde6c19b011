#!/usr/bin/env python
"""Soak test: many calls of mixed sizes and alphas through both entry points; device memory and host RSS must stay
flat, results must stay identical to the first pass.

    python tools/gpu_soak.py [rounds]
"""
import hashlib
import os
import resource
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1908_05944_b200 as ax  # noqa: E402
from paper_1908_05944_b200 import synth  # noqa: E402


def digest(k):
    h = hashlib.sha256()
    for a in (k.vertices, k.edges, k.triangles, k.tets):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(0)
    work = []
    for n in (1, 7, 300, 5_000, 40_000, 300_000, 1_000_000):
        c, r = synth.jittered_lattice(n, int(rng.integers(1 << 30)))
        for alpha in (0.0, 1.4):
            work.append((c, r, ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, 1e-300))))
    eng = ax.default_engine()
    first, mem0, rss0 = {}, None, None
    for it in range(rounds):
        for c, r, cfg in [work[i] for i in rng.permutation(len(work))]:
            key = (c.shape[0], cfg.alpha)
            k = ax.compute_alpha_complex_arrays(c, r, cfg)
            d = digest(k)
            outs = eng.compute_device(torch.as_tensor(c, device="cuda"), torch.as_tensor(r, device="cuda"), cfg)
            same_dev = all(np.array_equal(o.cpu().numpy(), a) for o, a in zip(outs, (k.vertices, k.edges, k.triangles, k.tets)))
            if first.setdefault(key, d) != d or not same_dev:
                print("MISMATCH", key, it, d, first[key], same_dev)
                sys.exit(1)
            del k, outs
        torch.cuda.synchronize()
        mem = torch.cuda.memory_allocated()
        rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
        if it == 2:
            mem0, rss0 = mem, rss
        if it % 10 == 0 or it == rounds - 1:
            print(f"round {it}: device allocated {mem / 2**20:.0f} MiB, host max RSS {rss / 2**10:.0f} MiB", flush=True)
    grew = (mem - mem0) / 2**20, (rss - rss0) / 2**10
    print(f"{rounds} rounds x {len(work)} workloads x 2 entry points: identical results; growth since round 2: "
          f"device {grew[0]:.0f} MiB, host max RSS {grew[1]:.0f} MiB")
    sys.exit(0 if grew[0] < 64 and grew[1] < 256 else 1)


if __name__ == "__main__":
    main()
