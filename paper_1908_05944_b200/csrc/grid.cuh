// grid.cuh -- validate_input + build_grid_arrays on the device
// (reference pipeline.py:224-245, grid.py:105-144).
//
// Counting sort by cell key: per-ball key + histogram (atomics), exclusive
// scan of the dense cell table, scatter, then a per-cell fix-up that orders
// the balls of one cell by ball index so the result equals the reference's
// stable argsort (grid.py:128).  The fix-up pass also writes the rank-space
// atom records and finds exact duplicate centres (they share a cell).
#pragma once

#include "common.cuh"
#include "predicates.cuh"

namespace axb {

constexpr int BOUNDS_THREADS = 256;

struct BoundsPartial {
    double lo[3], hi[3], rmax;
    unsigned int first_bad;
    unsigned int pad;
};

__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// grid.py:112, 119-120 (r_max, origin, span) + pipeline.py:235-237 (finite check).
// One partial per block; the last block to finish folds them (threadfence pattern).
__global__ void __launch_bounds__(BOUNDS_THREADS) k_bounds(const double *__restrict__ xyz,
                                                           const double *__restrict__ radii, int n,
                                                           BoundsPartial *__restrict__ partials,
                                                           unsigned int *__restrict__ done_counter,
                                                           BoundsPartial *__restrict__ result) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY}, rmax = -INFINITY;
    unsigned int bad = 0xffffffffu;
    // four balls per thread and step, their 16 loads issued before the first comparison
    const int stride = gridDim.x * blockDim.x;
    for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
        double x[4], y[4], z[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = min(i0 + u * stride, n - 1);        // clamped: a repeated ball changes nothing
            x[u] = xyz[3 * (size_t)i]; y[u] = xyz[3 * (size_t)i + 1]; z[u] = xyz[3 * (size_t)i + 2]; r[u] = radii[i];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = min(i0 + u * stride, n - 1);
            if (!(isfinite(x[u]) && isfinite(y[u]) && isfinite(z[u]) && isfinite(r[u]))) bad = min(bad, (unsigned)i);
            lo[0] = fmin(lo[0], x[u]); hi[0] = fmax(hi[0], x[u]);
            lo[1] = fmin(lo[1], y[u]); hi[1] = fmax(hi[1], y[u]);
            lo[2] = fmin(lo[2], z[u]); hi[2] = fmax(hi[2], z[u]);
            rmax = fmax(rmax, r[u]);
        }
    }
    __shared__ BoundsPartial s_part[BOUNDS_THREADS / 32];
    __shared__ bool s_last;
#pragma unroll
    for (int c = 0; c < 3; ++c) { lo[c] = warp_min_d(lo[c]); hi[c] = warp_max_d(hi[c]); }
    rmax = warp_max_d(rmax);
    bad = __reduce_min_sync(FULL, bad);
    int w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        for (int c = 0; c < 3; ++c) { s_part[w].lo[c] = lo[c]; s_part[w].hi[c] = hi[c]; }
        s_part[w].rmax = rmax;
        s_part[w].first_bad = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BoundsPartial p = s_part[0];
        for (int k = 1; k < BOUNDS_THREADS / 32; ++k) {
            for (int c = 0; c < 3; ++c) { p.lo[c] = fmin(p.lo[c], s_part[k].lo[c]); p.hi[c] = fmax(p.hi[c], s_part[k].hi[c]); }
            p.rmax = fmax(p.rmax, s_part[k].rmax);
            p.first_bad = min(p.first_bad, s_part[k].first_bad);
        }
        partials[blockIdx.x] = p;
        __threadfence();
        unsigned int ticket = atomicAdd(done_counter, 1u);
        s_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {
        // the last block folds all partials: threads stride over them, then the same two-level reduction
        __threadfence();
        const volatile BoundsPartial *vp = partials;
        double l2[3] = {INFINITY, INFINITY, INFINITY}, h2[3] = {-INFINITY, -INFINITY, -INFINITY}, rm = -INFINITY;
        unsigned int fb = 0xffffffffu;
        for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) {
            for (int c = 0; c < 3; ++c) { l2[c] = fmin(l2[c], vp[k].lo[c]); h2[c] = fmax(h2[c], vp[k].hi[c]); }
            rm = fmax(rm, vp[k].rmax);
            fb = min(fb, vp[k].first_bad);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) { l2[c] = warp_min_d(l2[c]); h2[c] = warp_max_d(h2[c]); }
        rm = warp_max_d(rm);
        fb = __reduce_min_sync(FULL, fb);
        __syncthreads();
        if (lane_id() == 0) {
            for (int c = 0; c < 3; ++c) { s_part[w].lo[c] = l2[c]; s_part[w].hi[c] = h2[c]; }
            s_part[w].rmax = rm;
            s_part[w].first_bad = fb;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            BoundsPartial p = s_part[0];
            for (int k = 1; k < BOUNDS_THREADS / 32; ++k) {
                for (int c = 0; c < 3; ++c) { p.lo[c] = fmin(p.lo[c], s_part[k].lo[c]); p.hi[c] = fmax(p.hi[c], s_part[k].hi[c]); }
                p.rmax = fmax(p.rmax, s_part[k].rmax);
                p.first_bad = min(p.first_bad, s_part[k].first_bad);
            }
            p.pad = 0;
            *result = p;
            *done_counter = 0;
        }
    }
}

// grid.py:122-127: clamped cell coordinates -> row-major key (x fastest); histogram.
__global__ void k_cell_keys(const double *__restrict__ xyz, GridView g, int *__restrict__ key_of_ball,
                            uint32_t *__restrict__ cell_count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    int cx = cell_coord(xyz[3 * (size_t)i], g.ox, g.side, g.dx);
    int cy = cell_coord(xyz[3 * (size_t)i + 1], g.oy, g.side, g.dy);
    int cz = cell_coord_z(xyz[3 * (size_t)i + 2], g);
    int key = cx + g.dx * (cy + g.dy * cz);
    key_of_ball[i] = key;
    atomicAdd(cell_count + key, 1u);
}

// scatter into cell ranges in arrival order; cell_count is consumed back to zero
__global__ void k_cell_scatter(int n, const int *__restrict__ key_of_ball, const uint32_t *__restrict__ cell_start,
                               uint32_t *__restrict__ cell_count, int *__restrict__ arrival) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int key = key_of_ball[i];
    unsigned slot = atomicSub(cell_count + key, 1u) - 1u;
    arrival[cell_start[key] + slot] = i;
}

// Per slot of the arrival order: final position inside the cell = number of
// cell mates with a smaller ball index (== stable sort by key, grid.py:128).
// Writes order/rank (grid.py:128-130), the rank-space atom record, reach
// (pipeline.py:322-324, -1 when not viable), and duplicate-centre records
// (pipeline.py:238-244: equal centres always share a cell).
__global__ void k_cell_finalize(int n, const double *__restrict__ xyz, const double *__restrict__ radii,
                                const int *__restrict__ key_of_ball, const uint32_t *__restrict__ cell_start,
                                const int *__restrict__ arrival, double alpha, double eps_abs,
                                int *__restrict__ orig_of_rank, int *__restrict__ rank_of_orig,
                                int4 *__restrict__ cell_of_rank, int dimx, int dimy, Atom *__restrict__ atoms, double *__restrict__ reach,
                                Atom *__restrict__ xyzr,
                                Counters *__restrict__ ctr, int2 *__restrict__ dup_records) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int i = arrival[t];
    int key = key_of_ball[i];
    int s = (int)cell_start[key], e = (int)cell_start[key + 1];
    double x = xyz[3 * (size_t)i], y = xyz[3 * (size_t)i + 1], z = xyz[3 * (size_t)i + 2];
    int pos = s;
    if (e - s > 1) {
        int dup = -1;
        for (int q = s; q < e; ++q) {
            int j = arrival[q];
            if (j < i) ++pos;
            else if (j > i && xyz[3 * (size_t)j] == x && xyz[3 * (size_t)j + 1] == y && xyz[3 * (size_t)j + 2] == z)
                dup = (dup < 0 || j < dup) ? j : dup;     // nearest later twin
        }
        if (dup >= 0) {
            unsigned slot = atomicAdd(&ctr->dup_count, 1u);
            if (slot < DUP_CAP) dup_records[slot] = make_int2(i, dup);
        }
    }
    double r = radii[i];
    double r2 = r * r;                                     // pipeline.py:590
    double lim = r2 + alpha + eps_abs;                     // pipeline.py:322
    Atom a;
    a.x = x; a.y = y; a.z = z; a.r2 = r2;
    atoms[pos] = a;
    const double rch = (lim >= 0.0) ? sqrt(fmax(lim, 0.0)) : -1.0;   // pipeline.py:323-324
    reach[pos] = rch;
    a.r2 = rch;                                            // (x, y, z, reach): one 32-byte load per edge candidate
    xyzr[pos] = a;
    orig_of_rank[pos] = i;
    rank_of_orig[i] = pos;
    const int rest = key / dimx;                           // (cx, cy, cz, key): k_edges wants the coordinates
    cell_of_rank[pos] = make_int4(key - rest * dimx, rest % dimy, rest / dimy, key);
}

__global__ void k_grid_export(int n, const int *__restrict__ orig_of_rank, const int *__restrict__ rank_of_orig,
                              const int *__restrict__ key_of_ball, int64_t *order, int64_t *rank, int64_t *cells) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (order) order[i] = orig_of_rank[i];
    if (rank) rank[i] = rank_of_orig[i];
    if (cells) cells[i] = key_of_ball[i];
}

}  // namespace axb
