"""Multi-GPU sharding of the hot path by grid slabs.

One process per GPU.  The GLOBAL grid geometry (reference grid.py:112-127) is
evaluated once on the host; ranks own contiguous z cell layers balanced by
atom count, load their layers plus a 2-layer halo on each side, and generate
exactly the simplices whose minimum-rank vertex they own -- the reference's
chunk ownership (pipeline.py:10-15: a chunk is a contiguous range of the
grid-sorted order, and z layers ARE contiguous rank ranges) mapped onto
GPUs.  Why 2 layers suffice with no exchange: every simplex incident to an
owned ball has all vertices within 2 cells of it, its ortho-centre within 1
cell, and the domination candidates within 1 cell of the centre
(pipeline.py:288-289, 316-320).  Like a reference chunk, a slab also emits the
faces its kept simplices inherit even when a neighbour owns them, so the
sorted duplicate-free union (pipeline.py:611-614) has to be taken across
slabs: rows are exchanged by owner-index range (one all_to_all), every rank
merges its range on its GPU, and the final gather of counts and rows to rank 0
is a concatenation in rank order.  (`ShardedJob.step(parallel_merge=False)`
keeps the simpler form: gather everything, merge on rank 0 alone.)

`local_compute` / `merge` are injectable so the plumbing is testable on CPU
with the gloo backend (tests/test_sharding.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

HALO_LAYERS = 2


@dataclass
class SlabPlan:
    origin: np.ndarray          # (3,) global grid origin
    cell_side: float
    dims: tuple                 # global (dx, dy, dz)
    layer: np.ndarray           # (n,) z cell layer of every ball
    owned: list                 # per rank: (z_own_lo, z_own_hi)
    rank_ranges: list           # per rank: (lo, hi) in the global grid-sorted order

    @property
    def world(self) -> int:
        return len(self.owned)


def plan_slabs(centers: np.ndarray, radii: np.ndarray, alpha: float, world: int) -> SlabPlan:
    """Global grid geometry + contiguous z-layer ownership balanced by atom count."""
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    n = centers.shape[0]
    if n == 0:
        raise ValueError("cannot shard an empty input")
    r_max = float(radii.max())
    side_sq = r_max * r_max + alpha                         # grid.py:112-113
    if side_sq <= 0.0:
        raise ValueError(f"alpha={alpha} gives non-positive squared cell side (r_max={r_max})")
    side = math.sqrt(side_sq)
    origin = centers.min(axis=0)
    span = centers.max(axis=0) - origin
    dims = tuple(int(d) for d in (np.floor(span / side).astype(np.int64) + 1))      # grid.py:121
    layer = np.clip(np.floor((centers[:, 2] - origin[2]) / side).astype(np.int64), 0, dims[2] - 1)   # grid.py:122-126
    hist = np.bincount(layer, minlength=dims[2])
    cum = np.concatenate([[0], np.cumsum(hist)])           # cum[z] = balls in layers < z = first grid rank of layer z
    cuts = [0]
    for r in range(1, world):
        z = int(np.searchsorted(cum, r * n / world, side="left"))
        cuts.append(min(max(z, cuts[-1]), dims[2]))
    cuts.append(dims[2])
    owned = [(cuts[r], cuts[r + 1]) for r in range(world)]
    rank_ranges = [(int(cum[a]), int(cum[b])) for a, b in owned]
    return SlabPlan(origin=origin, cell_side=side, dims=dims, layer=layer, owned=owned, rank_ranges=rank_ranges)


@dataclass
class SlabInput:
    centers: np.ndarray         # balls of the loaded layers, ascending global index
    radii: np.ndarray
    global_index: np.ndarray    # (n_local,) int64
    z_lo: int                   # loaded layers [z_lo, z_hi)
    z_hi: int
    z_own_lo: int
    z_own_hi: int


def slab_input(plan: SlabPlan, centers: np.ndarray, radii: np.ndarray, rank: int):
    """The balls rank `rank` loads (owned layers + halo), or None if it owns no layer."""
    own_lo, own_hi = plan.owned[rank]
    if own_lo >= own_hi:
        return None
    z_lo = max(own_lo - HALO_LAYERS, 0)
    z_hi = min(own_hi + HALO_LAYERS, plan.dims[2])
    gidx = np.flatnonzero((plan.layer >= z_lo) & (plan.layer < z_hi)).astype(np.int64)
    return SlabInput(centers=np.ascontiguousarray(centers[gidx]), radii=np.ascontiguousarray(radii[gidx]),
                     global_index=gidx, z_lo=z_lo, z_hi=z_hi, z_own_lo=own_lo, z_own_hi=own_hi)


def numpy_merge(parts: list, k: int) -> np.ndarray:
    """Sorted duplicate-free union of row lists (host stand-in for Engine.merge_rows in CPU tests)."""
    rows = [np.asarray(p, dtype=np.int64).reshape(-1, k) for p in parts]
    cat = np.concatenate(rows, axis=0) if rows else np.empty((0, k), dtype=np.int64)
    out = np.unique(cat, axis=0) if cat.shape[0] else cat
    return out.reshape(-1) if k == 1 else out


def gather_rows(local: list, dist, group=None, device="cpu", narrow: bool = False):
    """Gather the four row lists of every rank on rank 0: one all_gather of the counts, then every rank
    sends its exact rows (no padding) and rank 0 receives them straight into per-rank slices of ONE
    buffer per dimension, so the concatenation the merge needs already exists when the transfers end.
    `local` = [vertices (k0,), edges (k1,2), triangles (k2,3), tets (k3,4)] torch int64 tensors.
    narrow: the rows travel as int32 (the caller guarantees indices < 2^31) and rank 0 widens them back to the
    reference's int64 -- half the bytes into the one GPU everything converges on.
    Returns on rank 0: list over dims of (m_d, d+1) tensors (rank-major concatenation); elsewhere None."""
    import torch

    wire = torch.int32 if narrow else torch.int64
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = torch.tensor([int(t.shape[0]) for t in local], dtype=torch.int64, device=device)
    all_counts = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)           # the collective on counts
    all_counts = torch.stack(all_counts).cpu().numpy()         # (world, 4)
    # gloo (the CPU test / one-GPU developer transport) cannot send device memory: stage through the host there;
    # NCCL sends and receives the CUDA tensors directly over NVLink
    via_host = dist.get_backend(group) == "gloo" and str(device).startswith("cuda")
    tdev = "cpu" if via_host else device
    ops, bufs = [], []
    for d in range(4):
        width = d + 1
        mine = local[d].reshape(-1, width).contiguous().to(device=tdev, dtype=wire)
        if rank == 0:
            total = int(all_counts[:, d].sum())
            buf = torch.empty((total, width), dtype=wire, device=tdev)
            offs = np.concatenate([[0], np.cumsum(all_counts[:, d])]).astype(np.int64)
            buf[: mine.shape[0]] = mine
            for r in range(1, world):
                if all_counts[r, d]:
                    ops.append(dist.P2POp(dist.irecv, buf[int(offs[r]): int(offs[r + 1])], r, group))
            bufs.append(buf)
        elif mine.shape[0]:
            ops.append(dist.P2POp(dist.isend, mine, 0, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):                # the transfer of the rows (grouped NCCL send/recv)
            req.wait()
    if rank != 0:
        return None
    return [b.to(device=device, dtype=torch.int64) for b in bufs]


def exchange_by_owner(local: list, n_global: int, dist, group=None, device="cpu"):
    """Range-partitioned exchange: rank q becomes responsible for the rows whose first column (the owner =
    minimum ball index of the simplex) lies in [q * n / world, (q + 1) * n / world).  Every rank cuts its
    (canonical, hence owner-sorted) row lists at those boundaries and one all_to_all per dimension moves the
    pieces; afterwards each rank merges ITS range (1 / world of all rows) in parallel, and the final gather
    to rank 0 is a plain concatenation in rank order -- rank 0 no longer merges everything alone.
    `local` as in gather_rows.  Returns the four received row tensors (rank-major concatenation, unmerged)."""
    import torch

    world = dist.get_world_size(group)
    via_host = dist.get_backend(group) == "gloo" and str(device).startswith("cuda")
    tdev = "cpu" if via_host else device
    edges = torch.tensor([(q * n_global) // world for q in range(world + 1)], dtype=torch.int64, device=device)
    rows, send = [], []
    for d in range(4):
        r = local[d].reshape(-1, d + 1).contiguous()
        cut = torch.searchsorted(r[:, 0].contiguous(), edges)          # rows are sorted by owner
        cut[0], cut[-1] = 0, r.shape[0]
        rows.append(r)
        send.append(cut[1:] - cut[:-1])
    send_counts = torch.stack(send, dim=1).to(tdev).contiguous()         # (world, 4): rows for destination q, dimension d
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)        # the collective on counts
    send_np, recv_np = send_counts.cpu().numpy(), recv_counts.cpu().numpy()
    out = []
    for d in range(4):
        width = d + 1
        src = rows[d].to(tdev)
        dst = torch.empty((int(recv_np[:, d].sum()), width), dtype=torch.int64, device=tdev)
        dist.all_to_all_single(dst, src, output_split_sizes=[int(v) for v in recv_np[:, d]],
                               input_split_sizes=[int(v) for v in send_np[:, d]], group=group)   # the rows
        out.append(dst.to(device) if via_host else dst)
    return out


class ShardedJob:
    """One rank's share of a sharded run: owns the local inputs on its GPU; step() computes the
    slab, gathers everything on rank 0 and merges there."""

    def __init__(self, centers, radii, cfg, rank: int, world: int, engine, dist=None, group=None):
        import torch

        self.torch = torch
        self.cfg = cfg
        self.rank, self.world = rank, world
        self.engine = engine
        self.dist, self.group = dist, group
        self.n_global = int(np.asarray(radii).shape[0])
        self.plan = plan_slabs(centers, radii, cfg.alpha, world)
        self.slab = slab_input(self.plan, centers, radii, rank)
        dev = f"cuda:{engine.device}"
        self.device = dev
        if self.slab is not None:
            self.d_c = torch.as_tensor(self.slab.centers, device=dev)
            self.d_r = torch.as_tensor(self.slab.radii, device=dev)
            self.d_g = torch.as_tensor(self.slab.global_index, device=dev)

    @property
    def n_owned(self) -> int:
        lo, hi = self.plan.rank_ranges[self.rank]
        return hi - lo

    def local(self):
        torch = self.torch
        if self.slab is None:
            return [torch.empty((0,) if d == 0 else (0, d + 1), dtype=torch.int64, device=self.device) for d in range(4)]
        return self.engine.compute_slab_device(self.d_c, self.d_r, self.d_g, self.cfg, self.plan, self.slab)

    def step(self, parallel_merge: bool = True):
        """Returns the four merged CUDA tensors on rank 0, None elsewhere.
        parallel_merge: exchange rows by owner range, merge 1 / world of them on every rank, gather the sorted
        pieces (default); otherwise gather everything and merge on rank 0 alone."""
        outs = self.local()
        if self.world > 1 and parallel_merge:
            mine = exchange_by_owner(outs, self.n_global, self.dist, self.group, device=self.device)
            merged = [self.engine.merge_rows(mine[d], d + 1, self.n_global) for d in range(4)]
            parts = gather_rows(merged, self.dist, self.group, device=self.device, narrow=self.n_global < 2 ** 31)
            if parts is None:
                return None
            return [p.reshape(-1) if d == 0 else p for d, p in enumerate(parts)]     # owner ranges ascend with the rank
        if self.world == 1:
            parts = [[o] for o in outs]
        else:
            parts = gather_rows(outs, self.dist, self.group, device=self.device)
            if parts is None:
                return None
        torch = self.torch
        merged = []
        for d in range(4):
            cat = parts[d] if torch.is_tensor(parts[d]) else torch.cat([p.reshape(-1, d + 1) for p in parts[d]], dim=0)
            merged.append(self.engine.merge_rows(cat, d + 1, self.n_global))
        return merged


def compute_sharded_single_gpu(centers, radii, cfg, world: int, engine):
    """All `world` slabs one after the other on ONE GPU, then the merge: the sharded algorithm
    without the transport (used to validate slab ownership where only one GPU is available)."""
    import torch

    jobs = [ShardedJob(centers, radii, cfg, r, world, engine) for r in range(world)]
    per_rank = [j.local() for j in jobs]
    merged = []
    for d in range(4):
        cat = torch.cat([outs[d].reshape(-1, d + 1) for outs in per_rank], dim=0)
        merged.append(engine.merge_rows(cat, d + 1, len(radii)))
    return merged, per_rank
