"""The multi-GPU path as PROCESSES: `world` ranks, each with its own CUDA context, engine and slab, run
`ShardedJob.step()` -- `axb_compute_slab` through the C-ABI, the agreement on one status, the gather of
counts and rows to rank 0 and the merge there -- and the result must equal the single pass and the CPU
oracle bit for bit.  The box has one GPU, so every rank uses cuda:0 and the transport is gloo (NCCL
refuses two ranks on one device); with one GPU per rank the same code runs over NCCL (`bench.py --gpus N`).
Mirrors the reference's determinism contract: identical bytes for any worker / chunk split
(reference pkg/tests/test_acceptance.py:218-233, pipeline.py:597-614)."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1908_05944_b200 import synth

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    if name == "lattice_a0":
        return synth.jittered_lattice(80_000, 12) + (0.0, 1e-300)
    if name == "lattice_a14":
        return synth.jittered_lattice(40_000, 13) + (1.4, 1e-300)
    if name == "adversarial_shuffled":
        return synth.adversarial_density(60_000, 2, shuffle=True) + (0.0, 1e-300)
    raise KeyError(name)


def _worker(rank, world, port, out_dir, names):
    import torch
    import torch.distributed as dist

    import paper_1908_05944_b200 as ax
    from paper_1908_05944_b200.sharding import ShardedJob

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = ax.default_engine(0)
        for name in names:
            c, r, alpha, eps = _case(name)
            cfg = ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps))
            job = ShardedJob(c, r, cfg, rank, world, eng, dist)
            launches = eng.kernel_launches
            for parallel in (False, True):
                merged = job.step(parallel_merge=parallel)
                if rank == 0:
                    np.savez(os.path.join(out_dir, f"{name}_{int(parallel)}.npz"), *[m.cpu().numpy() for m in merged],
                             rows=job.last_gather["rows"])
                else:
                    assert merged is None
            assert eng.kernel_launches - launches >= 30          # this rank's CUDA kernels did run
            dist.barrier()
        # one rank's slab fails: every rank must raise the SAME exception instead of hanging in the gather
        c, r, alpha, eps = _case("lattice_a0")
        top = np.argsort(c[:, 2])[-30:]
        i, j = sorted((int(top[2]), int(top[11])))
        c = c.copy()
        c[j] = c[i]
        job = ShardedJob(c, r, ax.PipelineConfig(alpha=0.0), rank, world, eng, dist)
        try:
            job.step()
            msg = "no error"
        except ax.DuplicateCenter as e:
            msg = str(e)
        with open(os.path.join(out_dir, f"dup_{rank}.txt"), "w") as f:
            f.write(msg)
        with open(os.path.join(out_dir, f"dup_expected_{rank}.txt"), "w") as f:
            f.write(f"balls {i} and {j} share the center {tuple(float(v) for v in c[i])}")
        # with the default pivot threshold this input holds a singular tet solve: every rank must
        # name the simplex the reference names for the whole input
        c, r, alpha, _ = _case("lattice_a0")
        job = ShardedJob(c, r, ax.PipelineConfig(alpha=alpha), rank, world, eng, dist)
        try:
            job.step()
            msg = "no error"
        except ax.DegenerateSimplex as e:
            msg = " ".join(str(v) for v in e.vertices)
        with open(os.path.join(out_dir, f"deg_{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_processes_equal_single_pass_and_oracle(tmp_path, world):
    import torch.multiprocessing as mp

    import paper_1908_05944_b200 as ax

    names = ("lattice_a0", "lattice_a14", "adversarial_shuffled")
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), names), nprocs=world, join=True)
    eng = ax.default_engine()
    for name in names:
        c, r, alpha, eps = _case(name)
        single = eng.compute_host(c, r, ax.PipelineConfig(alpha=alpha, tolerance=ax.TolerancePolicy(1e-9, eps)))
        ref = oracle.compute(c, r, alpha, eps_singular=eps, threads=os.cpu_count(), chunk=4000)
        assert ref.status == oracle.OK
        for parallel in (0, 1):
            got = np.load(os.path.join(str(tmp_path), f"{name}_{parallel}.npz"))
            for d, want in enumerate((ref.vertices, ref.edges, ref.triangles, ref.tets)):
                rows = got[f"arr_{d}"]
                assert rows.dtype == np.int64
                assert np.array_equal(rows, want), (name, parallel, d)
                assert np.array_equal(rows, single[d]), (name, parallel, d)
            if not parallel:
                # the slabs' lists are disjoint: what the ranks sent adds up to the global counts
                assert [int(v) for v in got["rows"].sum(axis=0)] == [len(ref.vertices), len(ref.edges), len(ref.triangles), len(ref.tets)]
    c, r, alpha, _ = _case("lattice_a0")
    ref = oracle.compute(c, r, alpha, threads=os.cpu_count(), chunk=4000)
    assert ref.status == oracle.DEGENERATE
    for rank in range(world):
        assert open(tmp_path / f"dup_{rank}.txt").read() == open(tmp_path / f"dup_expected_{rank}.txt").read()
        assert open(tmp_path / f"deg_{rank}.txt").read() == " ".join(str(v) for v in ref.error_vertices)
