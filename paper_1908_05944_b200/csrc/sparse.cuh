// sparse.cuh -- grid binning when the dense cell table would be too large
// (widely spread inputs: the reference keeps only occupied cells, grid.py:38-39).
//
// Balls are sorted by their 64-bit cell key with a stable LSD radix sort
// (8 bits per pass, only as many passes as the key range needs).  Stability +
// the initial order 0..n-1 give exactly the reference's (cell key, ball index)
// order (grid.py:128).  Neighbourhood lookups then binary-search the sorted keys
// (predicates.cuh: row_range) instead of indexing a table.
#pragma once

#include "common.cuh"
#include "grid.cuh"
#include "predicates.cuh"

namespace axb {

constexpr int RS_WARPS = 4;             // warps per block, one chunk per warp
constexpr int RS_CHUNK = 2048;          // elements per chunk

// grid.py:122-127 with 64-bit keys
__global__ void k_cell_keys64(const double *__restrict__ xyz, GridView g, long long *__restrict__ key_of_ball,
                              long long *__restrict__ keys, int *__restrict__ vals) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const long long cx = cell_coord(xyz[3 * (size_t)i], g.ox, g.side, g.dx);
    const long long cy = cell_coord(xyz[3 * (size_t)i + 1], g.oy, g.side, g.dy);
    const long long cz = cell_coord_z(xyz[3 * (size_t)i + 2], g);
    const long long key = cx + (long long)g.dx * (cy + (long long)g.dy * cz);
    key_of_ball[i] = key;
    keys[i] = key;
    vals[i] = i;
}

// per-chunk digit histogram, laid out digit-major so that one exclusive scan yields, for every
// (digit, chunk), the number of elements that must precede it
__global__ void __launch_bounds__(RS_WARPS * 32) k_rs_hist(const long long *__restrict__ keys, int n, int shift,
                                                          int nchunks, uint32_t *__restrict__ hist) {
    __shared__ unsigned s_h[RS_WARPS][256];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int chunk = blockIdx.x * RS_WARPS + warp;
    for (int d = lane; d < 256; d += 32) s_h[warp][d] = 0u;
    __syncwarp();
    if (chunk < nchunks) {
        const int lo = chunk * RS_CHUNK, hi = min(lo + RS_CHUNK, n);
        for (int t = lo + lane; t < hi; t += 32) atomicAdd(&s_h[warp][(unsigned)((keys[t] >> shift) & 255)], 1u);
    }
    __syncwarp();
    if (chunk < nchunks)
        for (int d = lane; d < 256; d += 32) hist[(size_t)d * nchunks + chunk] = s_h[warp][d];
}

// stable scatter: a warp walks its chunk 32 elements at a time; lanes with equal digits are ordered
// by lane (match_any), the running per-digit offset lives in shared memory
__global__ void __launch_bounds__(RS_WARPS * 32) k_rs_scatter(const long long *__restrict__ keys_in,
                                                             const int *__restrict__ vals_in, int n, int shift, int nchunks,
                                                             const uint32_t *__restrict__ hist_pre,
                                                             long long *__restrict__ keys_out, int *__restrict__ vals_out) {
    __shared__ unsigned s_off[RS_WARPS][256];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int chunk = blockIdx.x * RS_WARPS + warp;
    if (chunk >= nchunks) return;
    for (int d = lane; d < 256; d += 32) s_off[warp][d] = hist_pre[(size_t)d * nchunks + chunk];
    __syncwarp();
    const int lo = chunk * RS_CHUNK, hi = min(lo + RS_CHUNK, n);
    for (int t0 = lo; t0 < hi; t0 += 32) {
        const int t = t0 + lane;
        const bool valid = t < hi;
        long long key = 0;
        int val = 0;
        unsigned d = 256u + (unsigned)lane;               // invalid lanes: unique pseudo-digits, match nobody
        if (valid) { key = keys_in[t]; val = vals_in[t]; d = (unsigned)((key >> shift) & 255); }
        const unsigned peers = __match_any_sync(FULL, d);
        const int rank = __popc(peers & lanemask_lt());
        unsigned base = 0;
        if (valid) base = s_off[warp][d];
        __syncwarp();
        if (valid && rank == 0) s_off[warp][d] = base + (unsigned)__popc(peers);
        __syncwarp();
        if (valid) { keys_out[base + rank] = key; vals_out[base + rank] = val; }
    }
}

// rank-space records from the sorted order (the sparse twin of k_cell_finalize); duplicate centres
// share a cell, i.e. a run of equal keys
__global__ void k_sparse_finalize(int n, const double *__restrict__ xyz, const double *__restrict__ radii,
                                  const long long *__restrict__ skeys, const int *__restrict__ order, GridView g,
                                  double alpha, double eps_abs, int *__restrict__ orig_of_rank,
                                  int *__restrict__ rank_of_orig, int4 *__restrict__ cell_of_rank,
                                  Atom *__restrict__ atoms, double *__restrict__ reach, Atom *__restrict__ xyzr,
                                  Counters *__restrict__ ctr, int2 *__restrict__ dup_records) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = order[t];
    const long long key = skeys[t];
    const double x = xyz[3 * (size_t)i], y = xyz[3 * (size_t)i + 1], z = xyz[3 * (size_t)i + 2];
    for (int q = t + 1; q < n && skeys[q] == key; ++q) {          // later cell mates have larger ball indices
        const int j = order[q];
        if (xyz[3 * (size_t)j] == x && xyz[3 * (size_t)j + 1] == y && xyz[3 * (size_t)j + 2] == z) {
            unsigned slot = atomicAdd(&ctr->dup_count, 1u);
            if (slot < DUP_CAP) dup_records[slot] = make_int2(i, j);
            break;                                                 // nearest later twin only
        }
    }
    const double r = radii[i];
    const double r2 = r * r;
    const double lim = r2 + alpha + eps_abs;
    Atom a;
    a.x = x; a.y = y; a.z = z; a.r2 = r2;
    atoms[t] = a;
    const double rch = (lim >= 0.0) ? sqrt(fmax(lim, 0.0)) : -1.0;
    reach[t] = rch;
    a.r2 = rch;
    xyzr[t] = a;
    orig_of_rank[t] = i;
    rank_of_orig[i] = t;
    const long long rest = key / g.dx;
    cell_of_rank[t] = make_int4((int)(key - rest * g.dx), (int)(rest % g.dy), (int)(rest / g.dy), 0);
}

__global__ void k_grid_export64(int n, const int *__restrict__ orig_of_rank, const int *__restrict__ rank_of_orig,
                                const long long *__restrict__ key_of_ball, int64_t *order, int64_t *rank, int64_t *cells) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (order) order[i] = orig_of_rank[i];
    if (rank) rank[i] = rank_of_orig[i];
    if (cells) cells[i] = key_of_ball[i];
}

}  // namespace axb
