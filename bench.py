#!/usr/bin/env python
"""Benchmark of the alpha-complex hot path (BASELINE.json metric: alpha-complex
atoms/sec on B200, % of HBM roofline, CPU reference beside it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--atoms-per-gpu M] [--alpha A]

One "step" = one full pass of the hot path (grid binning -> potential edges /
triangles / tets -> pruning -> canonical int64 simplex lists) over one
synthetic protein-density point set (generator G2 of SURVEY.md 8(d)).

Workload at N=1: SURVEY.md 8(d) config 3 -- 1,000,000 atoms, seed 0, alpha 0.
At N>1 every rank owns one z-slab of 1,000,000 atoms of an N x 1,000,000-atom
set (weak scaling; N=8 is an 8M-atom assembly; `--atoms-per-gpu 1250000` gives
the 10M-atom config 4), halo atoms replicated; the slab kernels need no
collective, the union across slabs is one all_to_all of rows by owner range, a
parallel merge, and the final gather of counts and rows to rank 0.

Prints ONE JSON line (see the task contract): `value` = device-resident
throughput (inputs already in HBM, outputs left in HBM), `e2e` = the same
through the public host API with pinned host buffers (H2D + D2H inside the
timed region), `roofline` for the dominant kernel, `cpu_baseline` = the real
reference package (alphax 0.1.0, installed unmodified under baseline/_ref)
on all host cores over a bounded spatial sample of the workload, with its
parity digest against the GPU; `cpu_baseline_port` = the C/OpenMP port of the
same algorithm (oracle/) on the whole workload.  `--impl reference` times the
CPU implementation alone (the real package when importable, else the port).

`--gpus N` without a torchrun environment starts the N ranks itself (one
process per GPU, NCCL) and exits non-zero when the box has fewer than N
devices.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "alpha_complex_atoms_per_sec"
UNIT = "atoms/s"


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        try:
            return float(json.load(open(path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region.  The region lasts only tens of
    milliseconds, so NVML is polled from a thread every 5 ms (more often steals the GIL from the timed loop) (nvidia-smi -lms 200 would see
    nothing); nvidia-smi is the fallback when pynvml is missing."""

    REASONS = ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"), (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap"))

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.bits = 0
        self.max_mhz = None
        self.stop_flag = False
        self.thread = None
        self.how = "pynvml"

    def _handle(self, nv):
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def loop():
                while not self.stop_flag:
                    try:
                        self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        self.bits |= int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
        except Exception:
            self.how = "nvidia-smi"
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=10).stdout.strip().split(",")
                self.samples.append(float(out[0]))
                self.max_mhz = float(out[1])
            except Exception:
                self.how = "unavailable"

    def stop(self):
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=1)
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": [name for bit, name in self.REASONS if self.bits & bit],
                "source": self.how}


def algorithmic_bytes(n, G, E, T, Q, K):
    """compulsory traffic per stage (each distinct input read once, each output written
    once; fp64 coordinates/centres/sizes, int32 intermediate indices, int64 final rows)."""
    K0, K1, K2, K3 = K
    kept32 = 4 * K0 + 8 * K1 + 12 * K2 + 16 * K3
    kept64 = 2 * kept32
    S = {
        "grid": 32 * n + 32 * n + 8 * n + 4 * (G + 1),
        "potential_edges": 32 * n + 4 * G + 40 * E,
        "potential_triangles": (32 * n + 8 * E + 44 * T) + (32 * n + 8 * E + 12 * T + 48 * Q),   # fused with tets
        "prune_tets": 32 * n + 4 * G + 48 * Q + 16 * K3,
        "prune_triangles": 32 * n + 4 * G + 44 * T + 12 * K2,
        "prune_edges": 32 * n + 4 * G + 40 * E + 8 * K1,
        "prune_vertices": 32 * n + 4 * G + 4 * K0,
        "canonical": kept32 + kept32,
        "export": kept32 + kept64,
    }
    total = (S["grid"] + S["potential_edges"] + S["potential_triangles"]
             + (32 * n + 4 * G + 40 * E + 44 * T + 48 * Q + kept32) + kept32 + kept64)
    return S, total


KERNEL_OF_STAGE = {
    "grid": "k_bounds+k_cell_keys+scan+k_cell_scatter+k_cell_finalize",
    "potential_edges": "k_edges",
    "potential_triangles": "k_tri_tet3",
    "prune_tets": "k_prune_tets",
    "prune_triangles": "k_prune_tris",
    "prune_edges": "k_prune_edges",
    "prune_vertices": "k_prune_vertices",
    "canonical": "scan+k_scatter_edges_tris+k_scatter_tets",
    "export": "k_emit_edges+k_emit_tris+k_emit_tets+k_emit_vertices",
}


def make_workload(n_total, seed=0):
    from paper_1908_05944_b200 import synth

    return synth.jittered_lattice(n_total, seed)


def load_reference():
    """The unmodified reference package: `pip install --target baseline/_ref /root/reference/pkg` (git-ignored,
    travels to the GPU box with the snapshot) or wherever PYTHONPATH has it.  None if it is not importable."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "alphax")) and ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import alphax

        return alphax
    except Exception:
        return None


def spatial_sample(centers, radii, m):
    """The m atoms of the workload nearest (Chebyshev distance) to its centre: a cubic block of the SAME point set,
    so density, radii and neighbourhood sizes are the workload's (the reference's time is linear in n: log-log
    exponent 0.998, reference pkg/test_output.txt:45)."""
    n = len(radii)
    if m >= n:
        return centers, radii
    mid = 0.5 * (centers.min(axis=0) + centers.max(axis=0))
    d = np.abs(centers - mid).max(axis=1)
    keep = np.sort(np.argpartition(d, m)[:m])
    return np.ascontiguousarray(centers[keep]), np.ascontiguousarray(radii[keep])


def digest_rows(levels):
    import hashlib

    h = hashlib.sha256()
    for a in levels:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def run_real_reference(alphax, centers, radii, alpha, eps_sing, workers):
    """reference pkg/src/alphax/pipeline.py:571-628 through its public entry point, all host cores
    (workers = os.cpu_count(), chunk_size = n // (8 * cores))."""
    n = len(radii)
    balls = [alphax.Ball(tuple(float(v) for v in c), float(r), i) for i, (c, r) in enumerate(zip(centers, radii))]
    cfg = alphax.PipelineConfig(alpha=alpha, workers=workers, chunk_size=max(1, n // (8 * workers)),
                                tolerance=alphax.TolerancePolicy(1e-9, eps_sing))
    t0 = time.perf_counter()
    k = alphax.compute_alpha_complex(balls, cfg)
    dt = time.perf_counter() - t0
    return dt, (k.vertices, k.edges, k.triangles, k.tets)


def run_cpu(centers, radii, alpha, eps_sing, threads):
    import oracle

    n = len(radii)
    t0 = time.perf_counter()
    res = oracle.compute(centers, radii, alpha, eps_singular=eps_sing, threads=threads,
                         chunk=max(1, n // (8 * threads)))
    dt = time.perf_counter() - t0
    if res.status != oracle.OK:
        raise RuntimeError(f"oracle failed with status {res.status}")
    return dt, res


def bench_reference(args, rank, world):
    """The CPU implementation of the path on all host threads: the real reference package when it is importable
    (kind "reference"), else the C/OpenMP port of oracle/ (kind "port").  Each step is a bounded sample of the
    b200 arm's workload: the Python package needs ~1 min per million atoms and core, so a step is a cubic block of
    --sample-atoms atoms cut out of the same point set; the port is fast enough for the whole workload."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = args.atoms_per_gpu          # one GPU's share of the workload
    centers, radii = make_workload(n)
    alphax = None if args.cpu_kind == "port" else load_reference()
    if args.cpu_kind == "reference" and alphax is None:
        raise SystemExit("the reference package is not importable (baseline/_ref missing)")
    if alphax is not None:
        m = min(args.sample_atoms, n)
        sc, sr = spatial_sample(centers, radii, m)

        def one():
            return run_real_reference(alphax, sc, sr, args.alpha, args.eps_singular, threads)

        kind = "reference"
        sample = (f"alphax {alphax.__version__} compute_alpha_complex(workers={threads}, chunk_size={max(1, m // (8 * threads))}) on a "
                  f"cubic block of {m} atoms cut from the centre of the workload (G2 n={n} seed=0 alpha={args.alpha})")
    else:
        m = n

        def one():
            dt, res = run_cpu(centers, radii, args.alpha, args.eps_singular, threads)
            return dt, (res.vertices, res.edges, res.triangles, res.tets)

        kind = "port"
        sample = f"C/OpenMP port (oracle/), the whole workload: G2 n={n} seed=0 alpha={args.alpha}"
    for _ in range(min(args.warmup, 1)):
        one()
    times = []
    for _ in range(args.steps):
        dt, levels = one()
        times.append(dt)
    total = sum(times)
    value = m * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample + f", {args.steps} passes",
                         "sample_atoms": m, "sha256_rows": digest_rows(levels)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "simplices_per_sec": sum(int(np.asarray(a).shape[0]) for a in levels) * args.steps / total,
        "gpu_launches": 0,
    }
    if kind == "reference" and not args.no_port:
        # the port beside it, on the SAME sample (its result must be the reference's, bit for bit) and on the whole workload
        dt_s, res_s = run_cpu(sc, sr, args.alpha, args.eps_singular, threads)
        dt_w, _ = run_cpu(centers, radii, args.alpha, args.eps_singular, threads)
        line["cpu_baseline_port"] = {
            "value": n / dt_w, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"C/OpenMP port (oracle/), the whole workload once: {dt_w:.2f} s; the reference's sample once: {dt_s:.3f} s",
            "same_rows_as_reference_on_sample": digest_rows((res_s.vertices, res_s.edges, res_s.triangles, res_s.tets)) == line["cpu_baseline"]["sha256_rows"]}
    print(json.dumps(line))


def workload_config(args, n_local):
    return {"workload": f"SURVEY 8(d) config 3: G2 jittered lattice, {n_local} atoms per GPU, seed 0, "
                        f"1 atom/12 A^3, radii U[1.2,1.9] A, alpha={args.alpha} A^2",
            "atoms_per_gpu": n_local, "alpha": args.alpha, "eps_singular": args.eps_singular,
            "l2": "flushed (256 MiB write) between timed steps; per-step working set ~1.5 GB also exceeds L2",
            "sharding": ("one z-slab per rank, 2-cell halo replicated; every slab emits the simplices it generates (disjoint lists, no "
                         "cross-GPU dedup); rows redistributed by index range (all_to_all), interleaved on every rank, "
                         "gathered to rank 0 (NCCL send/recv)") if args.gpus > 1 else "single GPU"}


def bench_b200(args, rank, world, local_rank):
    import torch

    import paper_1908_05944_b200 as ax

    # developer hooks for a one-GPU box: AXB_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 and
    # AXB_BENCH_BACKEND=gloo replaces the transport (NCCL refuses two ranks on one device), so the whole
    # multi-rank path (slab planning, per-rank slabs, gather, merge) can be exercised and verified
    same_device = os.environ.get("AXB_BENCH_SAME_DEVICE") == "1"
    if same_device:
        local_rank = 0
    backend = os.environ.get("AXB_BENCH_BACKEND", "nccl")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (this package has no CPU fallback)")
    if not same_device and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py --gpus {world}: only {torch.cuda.device_count()} CUDA device(s) on this box")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist = dist_mod
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group(backend)
    eng = ax.default_engine(local_rank)
    tol = ax.TolerancePolicy(1e-9, args.eps_singular)
    cfg = ax.PipelineConfig(alpha=args.alpha, tolerance=tol)
    n = args.atoms_per_gpu

    job = None
    if world == 1:
        centers, radii = make_workload(n)
        n_total = n
    else:
        from paper_1908_05944_b200.sharding import ShardedJob

        n_total = n * world
        centers, radii = make_workload(n_total)
        job = ShardedJob(centers, radii, cfg, rank, world, eng, dist)
    if job is None:
        d_c = torch.as_tensor(centers, device="cuda")
        d_r = torch.as_tensor(radii, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def device_step():
        # N=1: the whole input on this GPU.  N>1: this rank's slab, then the gather + merge on rank 0.
        return eng.compute_device(d_c, d_r, cfg) if job is None else job.step()

    # ---- device-resident throughput
    for _ in range(args.warmup):
        outs = device_step()
    counts = tuple(int(o.shape[0]) for o in outs) if outs is not None else (0, 0, 0, 0)
    if args.verify and job is not None and rank == 0:
        # the merged complex of the sharded run against ONE unsharded pass over the whole input on this GPU
        whole = eng.compute_device(torch.as_tensor(centers, device="cuda"), torch.as_tensor(radii, device="cuda"), cfg)
        same = all(bool(torch.equal(a, b)) for a, b in zip(outs, whole))
        print(f"[verify] {world} slabs merged == single pass over {n_total} atoms: {same}", file=sys.stderr)
        if not same:
            raise SystemExit("sharded result differs from the single-pass result")
        del whole
    stage_acc = {}
    launches0 = eng.kernel_launches
    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()
    barrier()
    step_ms = []
    for _ in range(args.steps):
        flush.fill_(1)                      # evict L2 between timed iterations
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        outs = device_step()
        e1.record()
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    barrier()
    launches = eng.kernel_launches - launches0
    # The same K steps once more with the library's stage events on (axb_set_stage_timing): the per-stage / per-kernel
    # times the roofline uses.  They are off in the timed region above, as they are for any caller who does not ask for
    # stage_times (the ~30 event records of a run cost 0.04-0.06 ms); the clock sampler covers both regions.
    staged_ms = []
    with eng.timing_stages():
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            outs = device_step()
            e1.record()
            torch.cuda.synchronize()
            staged_ms.append(e0.elapsed_time(e1))
            for k, v in eng.last_stage_ms.items():
                stage_acc[k] = stage_acc.get(k, 0.0) + v
    barrier()
    clocks = sampler.stop() if rank == 0 else None
    dev_ms = float(sum(step_ms))
    if dist is not None:
        t = torch.tensor([dev_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    n_all, simplices_all = n_total, sum(counts)      # counts live on rank 0 (the merged complex)
    del outs

    # ---- end to end: pinned host inputs -> H2D -> hot path -> D2H of the int64 rows, every step
    if job is None:
        h_c = torch.as_tensor(centers).pin_memory()
        h_r = torch.as_tensor(radii).pin_memory()
        hc_np, hr_np = h_c.numpy(), h_r.numpy()
        h2d = int(hc_np.nbytes + hr_np.nbytes)

        def e2e_step():
            k = ax.compute_alpha_complex_arrays(hc_np, hr_np, cfg, device=local_rank)   # the public API call
            assert k.edges.dtype == np.int64 and k.tets.shape[1] == 4
            # bytes that actually crossed PCIe: the rows travel as int32 and host threads widen them to the
            # reference's int64 while later chunks are in flight (axb_compute_host_finish)
            return int(eng.lib.axb_last_d2h_bytes(eng.handle))
    else:
        slab = job.slab
        pins = [torch.as_tensor(a).pin_memory() for a in (slab.centers, slab.radii, slab.global_index)] if slab else []
        h2d = int(sum(p.numel() * p.element_size() for p in pins))

        def e2e_step():
            if slab is not None:
                job.d_c.copy_(pins[0], non_blocking=True)
                job.d_r.copy_(pins[1], non_blocking=True)
                job.d_g.copy_(pins[2], non_blocking=True)
            merged = job.step()
            if merged is None:
                return 0
            host = [torch.empty(m.shape, dtype=m.dtype, pin_memory=True).copy_(m, non_blocking=True) for m in merged]
            torch.cuda.synchronize()
            return sum(h.numel() * 8 for h in host)

    for _ in range(max(3, args.warmup)):          # (the third call of a problem shape is the first on remembered sizes)
        d2h = e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (CUDA-event stage times recorded inside the library)
    if job is not None:
        job.local()            # the merge on rank 0 dropped the slab state; redo the slab so its counts can be read
    pot = (C_int64 * 3)()
    eng.lib.axb_potential_counts(eng.handle, pot)
    info = ax._native.GridInfo()
    eng.lib.axb_grid_get_info(eng.handle, __import__("ctypes").byref(info))
    n_local = n if job is None else (len(job.slab.radii) if job.slab is not None else 0)
    S, b_total = algorithmic_bytes(n_local, int(info.n_cells), int(pot[0]), int(pot[1]), int(pot[2]), counts)
    stage_ms = {k: v / args.steps for k, v in stage_acc.items()}
    kernel_stages = [k for k in stage_ms if k in S and k not in ("grid", "canonical", "export")]
    top = max(kernel_stages, key=lambda k: stage_ms[k])
    peak, peak_src = measured_peak()
    achieved = S[top] / (stage_ms[top] * 1e-3) / 1e9
    # DRAM traffic and pipe utilisation of that kernel come from an ncu --set full capture of THIS workload committed
    # under profiles/ (a number taken under a profiler cannot be measured inside a timed run); the source is named
    traffic, traffic_source, secondary = None, None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(KERNEL_OF_STAGE[top])
            traffic_source = "profiles/traffic.json: " + tj.get("_note", "")
            secondary = tj.get("_pipes", {}).get(KERNEL_OF_STAGE[top])
        except Exception:
            traffic = None
    dram_frac = (traffic / (stage_ms[top] * 1e-3) / 1e9 / peak) if traffic else None
    ms_per_step = dev_ms / args.steps
    line = {
        "metric": METRIC, "value": n_all * args.steps / (dev_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, args.atoms_per_gpu),
        "simplices_per_sec": simplices_all * args.steps / (dev_ms * 1e-3),
        "counts": list(counts),
        "e2e": {"value": n_all * args.steps / e2e_s, "unit": UNIT, "ms_per_step": 1e3 * e2e_s / args.steps,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        # bound: the kernels move a few per cent of what HBM could deliver and keep the FP64 pipe 10-30 % busy: they are
        # bound by instruction issue / dependent latency, not by a roofline (`secondary` = ncu's pipe view of the kernel)
        "roofline": {"bound": "issue" if (dram_frac is not None and dram_frac < 0.10) else "hbm",
                     "kernel": KERNEL_OF_STAGE[top], "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_source,
                     "dram_frac_of_peak": dram_frac, "secondary": secondary, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(S[top]), "kernel_ms": stage_ms[top],
                     "kernel_ms_source": (f"CUDA events inside the library (axb_set_stage_timing) over a second pass of {args.steps} "
                                          f"steps on the same inputs, {sum(staged_ms) / args.steps:.4f} ms per step with the events; "
                                          "the timed region above runs without them, like any call that does not ask for stage_times"),
                     "pipeline": {"algorithmic_bytes": int(b_total), "bytes_per_atom": b_total / n,
                                  "achieved": b_total / (ms_per_step * 1e-3) / 1e9,
                                  "frac": b_total / (ms_per_step * 1e-3) / 1e9 / peak},
                     "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
                     "stage_gbs": {k: round(S[k] / (stage_ms[k] * 1e-3) / 1e9, 1) for k in S if stage_ms.get(k, 0) > 0}},
        "clocks": clocks,
    }
    if job is not None:
        g = job.last_gather
        line["collectives"] = {"backend": backend, "per_step": ["all_gather of 10 status words (agreement on one error)",
                                                                   "all_to_all of row counts + one all_to_all of rows per dimension (index ranges)",
                                                                   "all_gather of the 4 row counts", "grouped send/recv of the rows to rank 0"],
                               "rows_by_rank": g.get("rows").tolist() if g.get("rows") is not None else None,
                               "bytes_into_rank0_per_step": int(g.get("bytes", 0)), "wire": "int32" if n_total < 2 ** 31 else "int64"}
        if backend == "nccl":
            line["collectives"]["nccl_version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
    # ---- CPU baselines beside it (rank 0, N=1 only)
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        # (a) the C/OpenMP port on the whole workload, bit-exact check of the GPU result
        dt, res = run_cpu(centers, radii, args.alpha, args.eps_singular, threads)
        gpu_rows = eng.compute_host(centers, radii, cfg)
        same = all(np.array_equal(a, b) for a, b in zip(gpu_rows, (res.vertices, res.edges, res.triangles, res.tets)))
        port = {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"C/OpenMP port (oracle/), the whole step workload once ({n} atoms, alpha={args.alpha}): {dt:.2f} s",
                "gpu_output_bit_exact_with_cpu": bool(same)}
        # (b) the real reference package on a bounded sample, in its own process (its worker pool forks, which a
        # process with a CUDA context must not do); the GPU runs the same sample for the parity digest
        ref_line = None
        if load_reference() is not None:
            cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--cpu-kind", "reference", "--steps", "1",
                   "--warmup", "0", "--no-port", "--sample-atoms", str(args.cpu_sample_atoms), "--atoms-per-gpu", str(n),
                   "--alpha", str(args.alpha), "--eps-singular", str(args.eps_singular)]
            env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
                ref_line = json.loads(out.stdout.strip().splitlines()[-1])["cpu_baseline"]
            except Exception as exc:                      # keep the bench line; say what happened
                port["reference_unavailable"] = f"{type(exc).__name__}: {exc}"[:200]
        if ref_line is not None:
            sc, sr = spatial_sample(centers, radii, min(args.cpu_sample_atoms, n))
            ref_line["gpu_output_bit_exact_with_cpu"] = digest_rows(eng.compute_host(sc, sr, cfg)) == ref_line["sha256_rows"]
            line["cpu_baseline"] = ref_line
            line["cpu_baseline_port"] = port
        else:
            line["cpu_baseline"] = port
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def spawn_ranks(args):
    """`python bench.py --gpus N` from a plain shell: start the N ranks (one process per GPU) under torchrun."""
    import socket

    import torch

    same_device = os.environ.get("AXB_BENCH_SAME_DEVICE") == "1"
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if not same_device and have < args.gpus:
        print(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) on this box", file=sys.stderr)
        return 2
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 100; 3 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--atoms-per-gpu", type=int, default=1_000_000)
    ap.add_argument("--alpha", type=float, default=0.0)
    ap.add_argument("--eps-singular", type=float, default=1e-12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verify", action="store_true", help="N>1: check the merged complex against one unsharded pass on rank 0")
    ap.add_argument("--cpu-kind", default="auto", choices=["auto", "reference", "port"],
                    help="--impl reference: the real package (baseline/_ref), the C port, or the package when importable")
    ap.add_argument("--sample-atoms", type=int, default=50_000,
                    help="--impl reference with the real package: atoms per step (a cubic block of the workload)")
    ap.add_argument("--cpu-sample-atoms", type=int, default=200_000,
                    help="b200 arm: size of the sample the real reference is timed on beside the GPU (10-30 s of CPU work)")
    ap.add_argument("--no-port", action="store_true", help="--impl reference: skip the C port beside the real package")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 3 if args.impl == "reference" else 100      # a pass of the CPU implementation takes seconds
    if args.gpus > 1 and args.eps_singular == 1e-12:
        args.eps_singular = 1e-300          # multi-million-atom sets trip the default pivot threshold in BOTH
                                            # implementations; both arms of an N > 1 run use the same value
    if args.impl == "reference":
        bench_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} was started with WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")            # the communicator's own log (rings, NVLS) goes to stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    bench_b200(args, rank, world, local_rank)


from ctypes import c_int64 as C_int64  # noqa: E402

if __name__ == "__main__":
    main()
