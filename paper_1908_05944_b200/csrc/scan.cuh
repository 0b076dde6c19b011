// scan.cuh -- device-wide exclusive prefix sum over uint32: one launch, single pass with decoupled
// look-back (warp shuffles inside a tile; a tile is 1024 threads x 4 items).  Used for the
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

// ---- single pass with decoupled look-back over up to four equally long arrays (blockIdx.y = array): every tile
// publishes its aggregate, then sums the aggregates of its predecessors until it meets one whose inclusive prefix is
// already known, publishes its own inclusive prefix and writes its outputs -- each input is read once and each output
// written once (the three-launch form read the input twice and cost three launches per scan: six of the ~22 launches of
// a pass).  Tiles take their number from a ticket counter, so a tile's predecessors always run or have run.
struct Scan4 {
    const uint32_t *in[4];
    uint32_t *out[4];
    unsigned long long *status[4];   // per tile: state << 32 | value (0: nothing yet, 1: aggregate, 2: inclusive prefix)
    unsigned int *ticket;            // [4]
};

enum : unsigned long long { SCAN_AGG = 1ull << 32, SCAN_INCL = 2ull << 32 };

constexpr int LB_THREADS = 256;                       // look-back kernel: 256 threads x 16 items = the same 4096-element tile,
constexpr int LB_ITEMS = SCAN_TILE / LB_THREADS;      // but eight resident blocks per SM and 16-byte loads / stores

__global__ void __launch_bounds__(LB_THREADS) k_scan_lookback(Scan4 a, size_t n) {
    __shared__ unsigned s_warp[LB_THREADS / 32 + 1];
    __shared__ unsigned s_tile, s_prefix;
    const int arr = blockIdx.y;
    const uint32_t *in = a.in[arr];
    uint32_t *out = a.out[arr];
    unsigned long long *status = a.status[arr];
    const int lane = lane_id(), w = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket + arr, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const size_t base = (size_t)tile * SCAN_TILE + (size_t)threadIdx.x * LB_ITEMS;
    unsigned item[LB_ITEMS];
    if (base + LB_ITEMS <= n) {                              // whole run inside the array: four 16-byte loads
#pragma unroll
        for (int q = 0; q < LB_ITEMS / 4; ++q) {
            const uint4 v4 = *reinterpret_cast<const uint4 *>(in + base + 4 * q);
            item[4 * q] = v4.x; item[4 * q + 1] = v4.y; item[4 * q + 2] = v4.z; item[4 * q + 3] = v4.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < LB_ITEMS; ++i) item[i] = (base + i < n) ? in[base + i] : 0u;
    }
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < LB_ITEMS; ++i) v += item[i];
    // block scan: warp inclusive scans, then the eight warp totals by every thread
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += t;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    unsigned ex = x - v, total = 0;
#pragma unroll
    for (int k = 0; k < LB_THREADS / 32; ++k) {
        const unsigned t = s_warp[k];
        if (k < w) ex += t;
        total += t;
    }
    if (threadIdx.x == 0) {
        volatile unsigned long long *st = status;
        st[tile] = (tile == 0 ? SCAN_INCL : SCAN_AGG) | total;
        __threadfence();
    }
    if (w == 0) {                                            // warp 0 looks back, 32 predecessors at a time
        unsigned prefix = 0;
        if (tile > 0) {
            volatile unsigned long long *st = status;
            long long idx = (long long)tile - 1 - lane;
            for (;;) {
                unsigned long long sw = idx >= 0 ? st[idx] : SCAN_INCL;     // before the first tile: prefix 0, known
                while (__any_sync(FULL, (sw >> 32) == 0ull)) sw = idx >= 0 ? st[idx] : SCAN_INCL;
                const unsigned known = __ballot_sync(FULL, (sw >> 32) == 2ull);
                const int stop = known ? __ffs(known) - 1 : 32;             // nearest predecessor with an inclusive prefix
                unsigned add = lane <= stop ? (unsigned)(sw & 0xffffffffull) : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(FULL, add, o);
                prefix += add;
                if (known) break;
                idx -= 32;
            }
            if (lane == 0) {
                st[tile] = SCAN_INCL | (unsigned long long)(prefix + total);
                __threadfence();
            }
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    ex += s_prefix;
    if (base + LB_ITEMS <= n) {
#pragma unroll
        for (int q = 0; q < LB_ITEMS / 4; ++q) {
            uint4 o4;
            o4.x = ex; ex += item[4 * q];
            o4.y = ex; ex += item[4 * q + 1];
            o4.z = ex; ex += item[4 * q + 2];
            o4.w = ex; ex += item[4 * q + 3];
            *reinterpret_cast<uint4 *>(out + base + 4 * q) = o4;
        }
    } else {
#pragma unroll
        for (int i = 0; i < LB_ITEMS; ++i) {
            if (base + i < n) out[base + i] = ex;
            ex += item[i];
        }
    }
    if (base <= n && n < base + LB_ITEMS) out[n] = ex;       // items at and beyond n count as zero: ex is the grand total
                                                             // (the grid covers index n: ceil((n + 1) / SCAN_TILE) tiles)
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
