"""Host logic of the multi-GPU path on CPU: slab planning, halo selection, and the
gather + merge plumbing over torch.distributed (gloo, world_size 2).  Per-slab
results come from the CPU oracle's single-chunk pass (test infrastructure), so what
is under test is the sharding algebra: union over slabs == whole-input result."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1908_05944_b200 import sharding, synth


def arrays(res):
    return [res.vertices, res.edges, res.triangles, res.tets]


def test_plan_partitions_layers_and_ranks():
    c, r = synth.jittered_lattice(6000, 2)
    for world in (1, 2, 3, 8):
        plan = sharding.plan_slabs(c, r, 0.0, world)
        assert plan.owned[0][0] == 0 and plan.owned[-1][1] == plan.dims[2]
        for (a0, a1), (b0, b1) in zip(plan.owned, plan.owned[1:]):
            assert a1 == b0 and a0 <= a1
        assert plan.rank_ranges[0][0] == 0 and plan.rank_ranges[-1][1] == len(r)
        sizes = [hi - lo for lo, hi in plan.rank_ranges]
        assert sum(sizes) == len(r)
        if world > 1:
            assert max(sizes) < 2.0 * len(r) / world + plan_layer_max(plan)
        # geometry equals the reference grid's (pinned through the oracle)
        st, g = oracle.grid_build(c, r, 0.0)
        assert plan.cell_side == g.side and plan.dims == g.dims and np.array_equal(plan.origin, g.origin)
        # z layers are contiguous ranges of the grid order
        for (z0, z1), (lo, hi) in zip(plan.owned, plan.rank_ranges):
            owners = plan.layer[g.order[lo:hi]]
            assert owners.size == 0 or (owners.min() >= z0 and owners.max() < z1)


def plan_layer_max(plan):
    return int(np.bincount(plan.layer).max())


def test_halo_selection():
    c, r = synth.jittered_lattice(6000, 4)
    plan = sharding.plan_slabs(c, r, 1.4, 3)
    seen = np.zeros(len(r), dtype=int)
    for rank in range(3):
        s = sharding.slab_input(plan, c, r, rank)
        assert (np.diff(s.global_index) > 0).all()
        lay = plan.layer[s.global_index]
        assert lay.min() >= s.z_lo and lay.max() < s.z_hi
        assert s.z_lo == max(s.z_own_lo - 2, 0) and s.z_hi == min(s.z_own_hi + 2, plan.dims[2])
        assert np.array_equal(s.centers, c[s.global_index])
        seen[s.global_index[(lay >= s.z_own_lo) & (lay < s.z_own_hi)]] += 1
    assert (seen == 1).all()            # every ball is owned exactly once
    # more ranks than layers: surplus ranks own nothing
    tiny = sharding.plan_slabs(c[:50], r[:50], 0.0, 16)
    assert sum(1 for a, b in tiny.owned if a < b) <= tiny.dims[2]


def test_union_of_slab_chunks_is_the_complex():
    c, r = synth.jittered_lattice(4000, 7)
    for alpha in (0.0, 1.4):
        full = oracle.compute(c, r, alpha)
        plan = sharding.plan_slabs(c, r, alpha, 4)
        parts = [oracle.compute(c, r, alpha, rank_range=rr) for rr in plan.rank_ranges]
        for d in range(4):
            merged = sharding.numpy_merge([arrays(p)[d] for p in parts], d + 1)
            assert np.array_equal(merged, arrays(full)[d])
        # inherited faces really do cross slabs: the parts overlap
        assert sum(len(p.triangles) for p in parts) > len(full.triangles)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, r = synth.jittered_lattice(3000, 9)
        alpha = 0.6
        plan = sharding.plan_slabs(c, r, alpha, world)
        res = oracle.compute(c, r, alpha, rank_range=plan.rank_ranges[rank])
        local = [torch.as_tensor(a) for a in arrays(res)]
        gathered = sharding.gather_rows(local, dist, device="cpu")
        if rank == 0:
            merged = [sharding.numpy_merge([gathered[d].numpy()], d + 1) for d in range(4)]
            np.savez(os.path.join(out_dir, "merged.npz"), *merged)
        else:
            assert gathered is None
        # range-partitioned form: exchange by owner, merge the own range, gather the sorted pieces
        mine = sharding.exchange_by_owner(local, len(r), dist, device="cpu")
        lo, hi = rank * len(r) // world, (rank + 1) * len(r) // world
        own = []
        for d in range(4):
            rows = mine[d].numpy().reshape(-1, d + 1)
            assert rows.shape[0] == 0 or (rows[:, 0].min() >= lo and rows[:, 0].max() < hi)
            own.append(torch.as_tensor(sharding.numpy_merge([rows], d + 1)))
        pieces = sharding.gather_rows(own, dist, device="cpu")
        if rank == 0:
            np.savez(os.path.join(out_dir, "merged_parallel.npz"), *[p.numpy() for p in pieces])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_and_merge_over_gloo(tmp_path, world):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(os.path.join(str(tmp_path), "merged.npz"))
    c, r = synth.jittered_lattice(3000, 9)
    full = oracle.compute(c, r, 0.6)
    par = np.load(os.path.join(str(tmp_path), "merged_parallel.npz"))
    for d in range(4):
        assert np.array_equal(got[f"arr_{d}"], arrays(full)[d])
        assert np.array_equal(par[f"arr_{d}"].reshape(arrays(full)[d].shape), arrays(full)[d])
