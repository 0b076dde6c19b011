"""Host logic of the multi-GPU path on CPU: slab planning, halo selection, the agreement on one
status, and the gather + merge plumbing over torch.distributed (gloo, world_size 2 and 3).  Per-slab
rows are cut out of the CPU oracle's complex by generator rank (test infrastructure: exactly what a
slab must emit), so what is under test is the sharding algebra and the transport; the CUDA slabs
themselves are checked against the same cut in tests/test_gpu_parity.py and tests/test_gpu_sharded.py."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1908_05944_b200 import sharding, synth
from paper_1908_05944_b200.errors import DegenerateSimplex, DuplicateCenter, NonFiniteCoordinate

from helpers import rows_generated_in


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
    """The reference's own chunk semantics (a chunk also emits inherited faces, pipeline.py:501-513) over slab
    rank ranges: the union is the complex but the parts OVERLAP -- which is why the CUDA slabs settle inherited
    faces themselves and emit by generator, so that their lists are disjoint (next test)."""
    c, r = synth.jittered_lattice(4000, 7)
    for alpha in (0.0, 1.4):
        full = oracle.compute(c, r, alpha)
        plan = sharding.plan_slabs(c, r, alpha, 4)
        parts = [oracle.compute(c, r, alpha, rank_range=rr) for rr in plan.rank_ranges]
        for d in range(4):
            merged = sharding.numpy_merge([arrays(p)[d] for p in parts], d + 1)
            assert np.array_equal(merged, arrays(full)[d])
        assert sum(len(p.triangles) for p in parts) > len(full.triangles)


def test_generator_cut_partitions_the_complex():
    c, r = synth.adversarial_density(4000, 3, shuffle=True)
    full = oracle.compute(c, r, 0.5, eps_singular=1e-300)
    st, g = oracle.grid_build(c, r, 0.5)
    plan = sharding.plan_slabs(c, r, 0.5, 5)
    parts = [rows_generated_in(arrays(full), g.rank, lo, hi) for lo, hi in plan.rank_ranges]
    for d in range(4):
        assert sum(p[d].shape[0] for p in parts) == arrays(full)[d].shape[0]
        assert np.array_equal(sharding.numpy_merge([p[d] for p in parts], d + 1), arrays(full)[d])
        # every simplex of a slab's cut touches only loaded layers (owned + 2 halo layers each side)
        for rank, p in enumerate(parts):
            if p[d].size:
                lay = plan.layer[p[d].reshape(-1)]
                z0, z1 = plan.owned[rank]
                assert lay.min() >= z0 and lay.max() < z1 + sharding.HALO_LAYERS
    assert plan.layer_start[0] == 0 and plan.layer_start[-1] == len(r)
    s = sharding.slab_input(plan, c, r, 2)
    assert s.first_rank == plan.layer_start[s.z_lo]


def test_plan_validates_like_the_reference():
    c, r = synth.jittered_lattice(500, 1)
    bad = c.copy()
    bad[17, 1] = np.nan
    with pytest.raises(NonFiniteCoordinate, match="ball 17 is not finite"):
        sharding.plan_slabs(bad, r, 0.0, 2)
    rr = r.copy()
    rr[3] = np.inf
    with pytest.raises(NonFiniteCoordinate, match="ball 3 is not finite"):
        sharding.plan_slabs(c, rr, 0.0, 2)
    with pytest.raises(ValueError, match="non-positive squared cell side"):
        sharding.plan_slabs(c, r, -100.0, 2)
    with pytest.raises(ValueError):
        sharding.plan_slabs(c, r[:-1], 0.0, 2)


def test_pick_error_is_the_reference_order():
    E = sharding.SlabError
    dup_a = E(status=6, vertices=(5, 9), xyz=(1.0, 2.0, 3.0))
    dup_b = E(status=6, vertices=(2, 3), xyz=(1.0, 2.0, 2.5))
    deg_a = E(status=7, key=(1 << 60) | (700 << 29) | 3, vertices=(1, 2))
    deg_b = E(status=7, key=(1 << 60) | (650 << 29) | 9, vertices=(4, 8))
    deg_tri = E(status=7, key=(3 << 60) | (10 << 29), vertices=(0, 1, 2))
    limit = E(status=10, message="too dense")
    assert sharding.pick_error([None, None]) is None
    assert sharding.pick_error([None, E(0)]) is None
    assert sharding.pick_error([deg_a, dup_a, None, dup_b])[1] is dup_b          # validation comes before any solve
    assert sharding.pick_error([deg_a, deg_tri, deg_b]) == (2, deg_b)          # smallest (stage, rank, ordinal)
    assert sharding.pick_error([limit, None, deg_tri])[1] is deg_tri
    assert sharding.pick_error([None, limit])[0] == 1
    for rec in (dup_a, deg_a, limit):
        back = E.unpack(rec.pack())
        assert (back.status, back.key, back.vertices, back.xyz) == (rec.status, rec.key, rec.vertices, rec.xyz)


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
        st, g = oracle.grid_build(c, r, alpha)
        local = [torch.as_tensor(a) for a in rows_generated_in(arrays(oracle.compute(c, r, alpha)), g.rank,
                                                                 *plan.rank_ranges[rank])]
        # one status for all ranks: nobody failed -> None everywhere; one rank failed -> everyone learns which error
        assert sharding.agree_on_error(None, dist) is None
        mine = sharding.SlabError(status=7, key=(1 << 60) | ((100 - rank) << 29), vertices=(rank, rank + 5)) if rank else None
        hit = sharding.agree_on_error(mine, dist)
        assert hit[0] == world - 1 and hit[1].vertices == (world - 1, world + 4)
        stats = {}
        gathered = sharding.gather_rows(local, dist, device="cpu", stats=stats)
        assert stats["rows"].shape == (world, 4) and int(stats["rows"][rank, 1]) == local[1].shape[0]
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
