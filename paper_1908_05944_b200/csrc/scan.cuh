// scan.cuh -- device-wide exclusive prefix sum over uint32 (three launches:
// per-tile sums, scan of the tile sums by one block, per-tile rescan).  Warp
// shuffles inside a tile; a tile is 1024 threads x 4 items.  Used for the
// dense cell table (counting sort, reference grid.py:128-134) and for the
// per-owner offsets of the canonical output.
#pragma once

#include "common.cuh"

namespace axb {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ unsigned block_excl_scan_1024(unsigned v, unsigned *s_warp, unsigned &total) {
    // inclusive scan in the warp
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned t = __shfl_up_sync(FULL, x, o);
        if (lane_id() >= o) x += t;
    }
    int w = threadIdx.x >> 5;
    if (lane_id() == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned y = s_warp[lane_id()];
        unsigned z = y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned t = __shfl_up_sync(FULL, z, o);
            if (lane_id() >= o) z += t;
        }
        s_warp[lane_id()] = z - y;      // exclusive warp offsets
        if (lane_id() == 31) s_warp[32] = z;
    }
    __syncthreads();
    unsigned r = s_warp[w] + x - v;
    total = s_warp[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile_sums(const uint32_t *__restrict__ in, size_t n,
                                                                  uint32_t *__restrict__ tile_sums) {
    __shared__ unsigned s_warp[33];
    size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i)
        if (base + i < n) v += in[base + i];
    unsigned total;
    block_excl_scan_1024(v, s_warp, total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// one block; tile_sums[i] <- exclusive prefix; tile_sums[ntiles] <- grand total
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_of_sums(uint32_t *__restrict__ tile_sums, size_t ntiles) {
    __shared__ unsigned s_warp[33];
    unsigned carry = 0;
    for (size_t base = 0; base < ntiles; base += SCAN_THREADS) {
        size_t i = base + threadIdx.x;
        unsigned v = i < ntiles ? tile_sums[i] : 0u;
        unsigned total;
        unsigned ex = block_excl_scan_1024(v, s_warp, total);
        if (i < ntiles) tile_sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) tile_sums[ntiles] = carry;
}

// out[i] = exclusive prefix of in (may alias); out[n] = total
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(const uint32_t *in, size_t n,
                                                              const uint32_t *__restrict__ tile_sums, uint32_t *out) {
    __shared__ unsigned s_warp[33];
    size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    unsigned item[SCAN_ITEMS];
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        item[i] = (base + i < n) ? in[base + i] : 0u;
        v += item[i];
    }
    unsigned total;
    unsigned ex = block_excl_scan_1024(v, s_warp, total) + tile_sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += item[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_sums[gridDim.x];
}

// ---- the same three steps over up to four equally long arrays in one go (blockIdx.y = array): the canonical
// stage scans the per-owner counters of all four dimensions, and twelve tiny launches cost more than the work
struct Scan4 {
    const uint32_t *in[4];
    uint32_t *out[4];
    uint32_t *sums[4];       // (ntiles + 1) each
};

__global__ void __launch_bounds__(SCAN_THREADS) k_scan4_tile_sums(Scan4 a, size_t n) {
    __shared__ unsigned s_warp[33];
    const uint32_t *in = a.in[blockIdx.y];
    size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i)
        if (base + i < n) v += in[base + i];
    unsigned total;
    block_excl_scan_1024(v, s_warp, total);
    if (threadIdx.x == 0) a.sums[blockIdx.y][blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan4_of_sums(Scan4 a, size_t ntiles) {
    __shared__ unsigned s_warp[33];
    uint32_t *tile_sums = a.sums[blockIdx.x];
    unsigned carry = 0;
    for (size_t base = 0; base < ntiles; base += SCAN_THREADS) {
        size_t i = base + threadIdx.x;
        unsigned v = i < ntiles ? tile_sums[i] : 0u;
        unsigned total;
        unsigned ex = block_excl_scan_1024(v, s_warp, total);
        if (i < ntiles) tile_sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) tile_sums[ntiles] = carry;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan4_apply(Scan4 a, size_t n) {
    __shared__ unsigned s_warp[33];
    const uint32_t *in = a.in[blockIdx.y];
    uint32_t *out = a.out[blockIdx.y];
    const uint32_t *tile_sums = a.sums[blockIdx.y];
    size_t base = (size_t)blockIdx.x * SCAN_TILE + (size_t)threadIdx.x * SCAN_ITEMS;
    unsigned item[SCAN_ITEMS];
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        item[i] = (base + i < n) ? in[base + i] : 0u;
        v += item[i];
    }
    unsigned total;
    unsigned ex = block_excl_scan_1024(v, s_warp, total) + tile_sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += item[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_sums[gridDim.x];
}

// ---- small arrays (one protein: a few tiles) in ONE launch: a single block walks the tiles with a carry;
// blockIdx.x picks the array, so the four scans of the canonical stage are still one launch
constexpr size_t SCAN_SMALL_TILES = 4;

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_small(Scan4 a, size_t n) {
    __shared__ unsigned s_warp[33];
    const uint32_t *in = a.in[blockIdx.x];
    uint32_t *out = a.out[blockIdx.x];
    unsigned carry = 0;
    for (size_t tile = 0; tile < n; tile += SCAN_TILE) {
        const size_t base = tile + (size_t)threadIdx.x * SCAN_ITEMS;
        unsigned item[SCAN_ITEMS];
        unsigned v = 0;
#pragma unroll
        for (int i = 0; i < SCAN_ITEMS; ++i) {
            item[i] = (base + i < n) ? in[base + i] : 0u;
            v += item[i];
        }
        unsigned total;
        unsigned ex = block_excl_scan_1024(v, s_warp, total) + carry;     // ends with a barrier: `in` may alias `out`
#pragma unroll
        for (int i = 0; i < SCAN_ITEMS; ++i) {
            if (base + i < n) out[base + i] = ex;
            ex += item[i];
        }
        carry += total;
    }
    if (threadIdx.x == 0) out[n] = carry;
}

}  // namespace axb
