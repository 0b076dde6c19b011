#!/usr/bin/env python
"""What one rank of a sharded run does, timed on ONE GPU (the box has no second one): the slab of every rank of a
`world`-way job computed in turn (device time per slab), then the two ways of interleaving the slabs' disjoint row
lists -- all rows on one GPU (what rank 0 does when it merges alone) and 1 / world of them (what every rank does after
the index-range redistribution).  Transfers are not part of this; DESIGN.md section 6 adds them at NVLink rates.

    python tools/gpu_shard_probe.py [atoms_per_rank] [world ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_05944_b200 as ax
from paper_1908_05944_b200 import synth
from paper_1908_05944_b200.sharding import ShardedJob

per_rank = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
worlds = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
eng = ax.default_engine()
cfg = ax.PipelineConfig(alpha=0.0, tolerance=ax.TolerancePolicy(1e-9, 1e-300))


def timed(fn, reps=8):
    fn()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


for world in worlds:
    n = per_rank * world
    c, r = synth.jittered_lattice(n, 0)
    jobs = [ShardedJob(c, r, cfg, q, world, eng) for q in range(world)]
    slab_ms, outs = [], []
    for j in jobs:
        ms, o = timed(j.local)
        slab_ms.append(ms)
        outs.append([t.clone() for t in o])
    loaded = [int(j.slab.radii.shape[0]) for j in jobs]
    cat = [torch.cat([o[d].reshape(-1, d + 1) for o in outs]) for d in range(4)]
    merge_all_ms, merged = timed(lambda: [eng.merge_rows(cat[d], d + 1, n) for d in range(4)])
    # one rank's share after the redistribution: the rows whose first index falls into its range
    lo, hi = 0, n // world
    part = [t[(t.reshape(-1, d + 1)[:, 0] >= lo) & (t.reshape(-1, d + 1)[:, 0] < hi)] for d, t in enumerate(cat)]
    merge_part_ms, _ = timed(lambda: [eng.merge_rows(part[d], d + 1, hi, index_lo=lo) for d in range(4)])
    rows = [int(m.shape[0]) for m in merged]
    wire = sum(int(o[d].numel()) for o in outs[1:] for d in range(4)) * 4
    print(json.dumps({"world": world, "atoms": n, "loaded_per_rank": loaded, "slab_ms": [round(v, 3) for v in slab_ms],
                      "merge_all_on_one_gpu_ms": round(merge_all_ms, 3), "merge_one_share_ms": round(merge_part_ms, 3),
                      "rows": rows, "int32_bytes_into_rank0": wire}))
