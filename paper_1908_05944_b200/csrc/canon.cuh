// canon.cuh -- canonical sort + dedup of the kept simplices
// (reference pipeline.py:611-614 via _arrays.py:12-16: rows of ascending ball
// indices, lexicographically sorted, duplicate-free, int64).
//
// No global sort: a canonical row starts with its minimum ball index, so rows
// are bucketed by that "owner".  Bucket sizes were counted while pruning;
// an exclusive scan turns them into the final row offsets, a scatter drops
// every kept simplex into its owner's bucket, and a rank-sort inside the
// (tiny) bucket writes the int64 rows straight to their final position.
// Each simplex is represented exactly once (a kept-bit / kept-flag / kept-list
// entry), so there is nothing to deduplicate; an equal pair inside a bucket
// would be a logic error and is reported.
#pragma once

#include "common.cuh"

namespace axb {

struct CanonParams {
    int n;
    const int *orig;
    const uint32_t *adj_off;
    const int *pe_u;
    const int *pe_v;
    uint32_t pe_cap;
    int W;
    const unsigned long long *trimask;
    const unsigned int *eflag;
    const int4 *k3;
    uint32_t *cnt1, *cnt2, *cnt3;          // consumed as cursors
    const uint32_t *off1, *off2, *off3;    // (n + 1) exclusive offsets per owner
    int2 *tmp1;                            // (owner, b)
    int4 *tmp2;                            // (owner, b, c, -)
    int4 *tmp3;                            // (owner, b, c, d)
    Counters *ctr;
    int own_lo, own_hi;                    // rows of generators outside [own_lo, own_hi) are not emitted (slab ownership)
};

__device__ __forceinline__ bool canon_emits(const CanonParams &P, int gen) { return gen >= P.own_lo && gen < P.own_hi; }

// cap1 / cap2: capacities of the bucket arrays (they are sized from the exact counts, or -- axb_compute_into -- from
// what the caller's buffers hold, before the counts are known on the host)
#ifndef SCATTER_MLP
#define SCATTER_MLP 1
#endif
__device__ __forceinline__ void scatter_tets_rows(const CanonParams &P, unsigned k3_cap, unsigned cap3) {
    const unsigned n_k3 = min(P.ctr->n_k3, k3_cap);
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n_k3; e += gridDim.x * blockDim.x) {
        const int4 r = P.k3[e];
        const unsigned pos = P.off3[r.x] + atomicSub(P.cnt3 + r.x, 1u) - 1u;
        if (pos < cap3) P.tmp3[pos] = r;
    }
}

// (launched with gridDim.y == 2, the second layer of blocks drops the kept tets into their buckets: one launch for the
// three lists; k3_cap / cap3 are ignored otherwise)
__global__ void __launch_bounds__(256) k_scatter_edges_tris(CanonParams P, unsigned cap1, unsigned cap2, unsigned k3_cap = 0,
                                                            unsigned cap3 = 0) {
    if (blockIdx.y == 1) { scatter_tets_rows(P, k3_cap, cap3); return; }
    if (P.ctr->n_pe > P.pe_cap) return;      // the edge list overflowed its buffer (only a run on remembered sizes gets this
                                             // far: its tail was never written; the host redoes the run after its final sync)
    const unsigned n_pe = P.ctr->n_pe;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n_pe; e += gridDim.x * blockDim.x) {
        const int u = __ldg(P.pe_u + e), v = __ldg(P.pe_v + e);
        if (!canon_emits(P, u)) continue;
#if SCATTER_MLP
        // A warp issues in order, so every level of the dependent chain (list entry -> ball indices -> bucket slot -> row)
        // is issued for the edge AND up to three triangles of its row before anything waits for the previous level:
        // the chain is six round trips deep whatever the row holds (it was four per triangle on top of the edge's four).
        if (P.W == 1) {
            unsigned flag = P.eflag[e];
            unsigned long long m = P.trimask[e];
            if (!flag && !m) continue;
            const int ou = __ldg(P.orig + u), ov = __ldg(P.orig + v);
            const unsigned bu = __ldg(P.adj_off + u);
            const int ea = min(ou, ov), eb = max(ou, ov);
            do {
                int j[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    j[k] = -1;
                    if (m) { j[k] = __ffsll((long long)m) - 1; m &= m - 1; }
                }
                int pw[3], ow[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) pw[k] = j[k] >= 0 ? __ldg(P.pe_v + bu + j[k]) : 0;
#pragma unroll
                for (int k = 0; k < 3; ++k) ow[k] = j[k] >= 0 ? __ldg(P.orig + pw[k]) : 0;
                // owners, bucket offsets and slots: every load and atomic issued before the first result is needed
                unsigned es = 0, eo = 0;
                if (flag) { eo = P.off1[ea]; es = atomicSub(P.cnt1 + ea, 1u); }
                int ta[3], tb[3], tc[3];
                unsigned tsl[3], to[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    int a = ou, b = ov, c = ow[k], t;
                    if (a > b) { t = a; a = b; b = t; }
                    if (b > c) { t = b; b = c; c = t; }
                    if (a > b) { t = a; a = b; b = t; }
                    ta[k] = a; tb[k] = b; tc[k] = c;
                    tsl[k] = 0; to[k] = 0;
                    if (j[k] >= 0) { to[k] = P.off2[a]; tsl[k] = atomicSub(P.cnt2 + a, 1u); }
                }
                if (flag) {
                    const unsigned pos = eo + es - 1u;
                    if (pos < cap1) P.tmp1[pos] = make_int2(ea, eb);
                }
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    if (j[k] >= 0) {
                        const unsigned pos = to[k] + tsl[k] - 1u;
                        if (pos < cap2) P.tmp2[pos] = make_int4(ta[k], tb[k], tc[k], 0);
                    }
                flag = 0u;                  // (more than three triangles in the row: another round, without the edge)
            } while (m);
            continue;
        }
#endif
        const int ou = __ldg(P.orig + u), ov = __ldg(P.orig + v);
        if (P.eflag[e]) {
            const int a = min(ou, ov), b = max(ou, ov);
            const unsigned pos = P.off1[a] + atomicSub(P.cnt1 + a, 1u) - 1u;
            if (pos < cap1) P.tmp1[pos] = make_int2(a, b);
        }
        const unsigned bu = __ldg(P.adj_off + u);
        for (int w = 0; w < P.W; ++w) {
            unsigned long long m = P.trimask[(size_t)e * P.W + w];
            while (m) {
                const int j = 64 * w + __ffsll((long long)m) - 1;
                m &= m - 1;
                const int ow = __ldg(P.orig + __ldg(P.pe_v + bu + j));
                int a = ou, b = ov, c = ow, t;
                if (a > b) { t = a; a = b; b = t; }
                if (b > c) { t = b; b = c; c = t; }
                if (a > b) { t = a; a = b; b = t; }
                const unsigned pos = P.off2[a] + atomicSub(P.cnt2 + a, 1u) - 1u;
                if (pos < cap2) P.tmp2[pos] = make_int4(a, b, c, 0);
            }
        }
    }
}

// one dimension at a time (the pipelined host path canonicalises a dimension as soon as it is final);
// `cap` guards the bucket array, whose size was fixed before the exact count was known
__global__ void __launch_bounds__(256) k_scatter_edges(CanonParams P, unsigned cap) {
    if (P.ctr->n_pe > P.pe_cap) return;      // the edge list overflowed its buffer (only a run on remembered sizes gets this
                                             // far: its tail was never written; the host redoes the run after its final sync)
    const unsigned n_pe = P.ctr->n_pe;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n_pe; e += gridDim.x * blockDim.x) {
        if (!P.eflag[e]) continue;
        const int u = __ldg(P.pe_u + e);
        if (!canon_emits(P, u)) continue;
        const int ou = __ldg(P.orig + u), ov = __ldg(P.orig + __ldg(P.pe_v + e));
        const int a = min(ou, ov), b = max(ou, ov);
        const unsigned pos = P.off1[a] + atomicSub(P.cnt1 + a, 1u) - 1u;
        if (pos < cap) P.tmp1[pos] = make_int2(a, b);
    }
}

__global__ void __launch_bounds__(256) k_scatter_tris(CanonParams P, unsigned cap) {
    if (P.ctr->n_pe > P.pe_cap) return;      // the edge list overflowed its buffer (only a run on remembered sizes gets this
                                             // far: its tail was never written; the host redoes the run after its final sync)
    const unsigned n_pe = P.ctr->n_pe;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n_pe; e += gridDim.x * blockDim.x) {
        unsigned long long any = 0ull;
        for (int w = 0; w < P.W; ++w) any |= P.trimask[(size_t)e * P.W + w];
        if (!any) continue;
        const int u = __ldg(P.pe_u + e);
        if (!canon_emits(P, u)) continue;
        const int ou = __ldg(P.orig + u), ov = __ldg(P.orig + __ldg(P.pe_v + e));
        const unsigned bu = __ldg(P.adj_off + u);
#if SCATTER_MLP
        if (P.W == 1) {         // level by level for up to three triangles of the row (see k_scatter_edges_tris)
            unsigned long long m = any;
            do {
                int j[3], pw[3], ow[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    j[k] = -1;
                    if (m) { j[k] = __ffsll((long long)m) - 1; m &= m - 1; }
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) pw[k] = j[k] >= 0 ? __ldg(P.pe_v + bu + j[k]) : 0;
#pragma unroll
                for (int k = 0; k < 3; ++k) ow[k] = j[k] >= 0 ? __ldg(P.orig + pw[k]) : 0;
                int ta[3], tb[3], tc[3];
                unsigned tsl[3], to[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    int a = ou, b = ov, c = ow[k], t;
                    if (a > b) { t = a; a = b; b = t; }
                    if (b > c) { t = b; b = c; c = t; }
                    if (a > b) { t = a; a = b; b = t; }
                    ta[k] = a; tb[k] = b; tc[k] = c;
                    tsl[k] = 0; to[k] = 0;
                    if (j[k] >= 0) { to[k] = P.off2[a]; tsl[k] = atomicSub(P.cnt2 + a, 1u); }
                }
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    if (j[k] >= 0) {
                        const unsigned pos = to[k] + tsl[k] - 1u;
                        if (pos < cap) P.tmp2[pos] = make_int4(ta[k], tb[k], tc[k], 0);
                    }
            } while (m);
            continue;
        }
#endif
        for (int w = 0; w < P.W; ++w) {
            unsigned long long m = P.trimask[(size_t)e * P.W + w];
            while (m) {
                const int j = 64 * w + __ffsll((long long)m) - 1;
                m &= m - 1;
                const int ow = __ldg(P.orig + __ldg(P.pe_v + bu + j));
                int a = ou, b = ov, c = ow, t;
                if (a > b) { t = a; a = b; b = t; }
                if (b > c) { t = b; b = c; c = t; }
                if (a > b) { t = a; a = b; b = t; }
                const unsigned pos = P.off2[a] + atomicSub(P.cnt2 + a, 1u) - 1u;
                if (pos < cap) P.tmp2[pos] = make_int4(a, b, c, 0);
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_scatter_tets(CanonParams P, unsigned k3_cap, unsigned cap3) {
    scatter_tets_rows(P, k3_cap, cap3);
}

// One thread per bucket entry: its position inside the bucket is the number of
// smaller entries; write the int64 row there.
// `map` (optional) renames local ball indices to global ones; it is ascending, so order is preserved.
__device__ __forceinline__ int64_t mapped(const int64_t *__restrict__ map, int v) { return map ? map[v] : (int64_t)v; }

// Row writers.  PlainOut<int64_t>: the reference dtype (device-resident results).  PlainOut<int32_t>: the host
// path -- half the PCIe bytes, widened to int64 by host threads while the next chunk is in flight.  Packed24Out:
// the host path while ball indices fit 24 bits -- three bytes per value.  The value stream is cut into chunks of
// whole rows (one D2H copy each); a chunk of m values is stored as m low halves (uint16) followed by m
// high bytes, so both planes stay aligned and the host unpacks them with plain vector loads (widen_pool.h).
template <class T>
struct PlainOut {
    T *p;
    struct Row {
        T *q;
        __device__ __forceinline__ void put(int c, int64_t v) const { q[c] = (T)v; }
    };
    __device__ __forceinline__ Row row(size_t pos, size_t, int K) const { return Row{p + (size_t)K * pos}; }
};
struct Packed24Out {
    unsigned char *p;
    unsigned rows_shift;          // a chunk holds 1 << rows_shift whole rows (so a row never straddles two chunks)
    struct Row {
        unsigned short *lo;
        unsigned char *hi;
        __device__ __forceinline__ void put(int c, int64_t v) const {
            lo[c] = (unsigned short)(v & 0xffff);
            hi[c] = (unsigned char)(v >> 16);
        }
    };
    __device__ __forceinline__ Row row(size_t pos, size_t total_rows, int K) const {
        const size_t first = pos >> rows_shift << rows_shift;              // all chunks before this one are full
        const size_t m = min((size_t)1 << rows_shift, total_rows - first) * (size_t)K;     // values in this chunk
        unsigned char *b = p + first * (size_t)K * 3;
        const size_t within = (pos - first) * (size_t)K;
        return Row{reinterpret_cast<unsigned short *>(b) + within, b + 2 * m + within};
    }
};

// `total_dev` (optional) = device-side row count (the last entry of the offset array): lets the caller
// launch without knowing the count on the host; `total` then carries the capacity the buffers were sized for.
// SKIP0: write only the columns after the owner (the host rebuilds column 0 from the offsets)
template <class Out, bool SKIP0 = false>
__device__ __forceinline__ void emit_edges_rows(const int2 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                                unsigned total, const uint32_t *__restrict__ total_dev,
                                                const int64_t *__restrict__ map, Out out, Counters *ctr) {
    if (total_dev) {                        // device-side row count; `total` then is the CAPACITY of tmp / out: when the
        const unsigned cap = total;         // count exceeds it the host falls back (AXB_ERR_STATE) and nothing is read
        total = *total_dev;
        if (total > cap) return;
    }
    for (unsigned s = blockIdx.x * blockDim.x + threadIdx.x; s < total; s += gridDim.x * blockDim.x) {
    const int2 me = tmp[s];
    const unsigned lo = off[me.x], hi = off[me.x + 1];
    unsigned pos = lo;
    for (unsigned q = lo; q < hi; ++q) {
        const int b = tmp[q].y;
        if (b < me.y) ++pos;
        else if (b == me.y && q != s) atomicOr(&ctr->overflow, 1u << 5);
    }
    if (SKIP0) {
        out.row(pos, total, 1).put(0, mapped(map, me.y));
    } else {
        const auto w = out.row(pos, total, 2);
        w.put(0, mapped(map, me.x));
        w.put(1, mapped(map, me.y));
    }
    }
}

template <class Out, bool SKIP0 = false>
__global__ void __launch_bounds__(256) k_emit_edges(const int2 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                                    unsigned total, const uint32_t *__restrict__ total_dev,
                                                    const int64_t *__restrict__ map, Out out, Counters *ctr) {
    emit_edges_rows<Out, SKIP0>(tmp, off, total, total_dev, map, out, ctr);
}

template <class Out, bool SKIP0 = false>
__device__ __forceinline__ void emit_tris_rows(const int4 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                               unsigned total, const uint32_t *__restrict__ total_dev,
                                               const int64_t *__restrict__ map, Out out, Counters *ctr) {
    if (total_dev) {                        // device-side row count; `total` then is the CAPACITY of tmp / out: when the
        const unsigned cap = total;         // count exceeds it the host falls back (AXB_ERR_STATE) and nothing is read
        total = *total_dev;
        if (total > cap) return;
    }
    for (unsigned s = blockIdx.x * blockDim.x + threadIdx.x; s < total; s += gridDim.x * blockDim.x) {
    const int4 me = tmp[s];
    const unsigned lo = off[me.x], hi = off[me.x + 1];
    unsigned pos = lo;
    for (unsigned q = lo; q < hi; ++q) {
        const int4 o = tmp[q];
        if (o.y < me.y || (o.y == me.y && o.z < me.z)) ++pos;
        else if (o.y == me.y && o.z == me.z && q != s) atomicOr(&ctr->overflow, 1u << 5);
    }
    if (SKIP0) {
        const auto w = out.row(pos, total, 2);
        w.put(0, mapped(map, me.y));
        w.put(1, mapped(map, me.z));
    } else {
        const auto w = out.row(pos, total, 3);
        w.put(0, mapped(map, me.x));
        w.put(1, mapped(map, me.y));
        w.put(2, mapped(map, me.z));
    }
    }
}

template <class Out, bool SKIP0 = false>
__global__ void __launch_bounds__(256) k_emit_tris(const int4 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                                   unsigned total, const uint32_t *__restrict__ total_dev,
                                                   const int64_t *__restrict__ map, Out out, Counters *ctr) {
    emit_tris_rows<Out, SKIP0>(tmp, off, total, total_dev, map, out, ctr);
}

template <class Out>
__device__ __forceinline__ void emit_tets_rows(const int4 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                               unsigned total, const uint32_t *__restrict__ total_dev,
                                               const int64_t *__restrict__ map, Out out, Counters *ctr) {
    if (total_dev) {                        // device-side row count; `total` then is the CAPACITY of tmp / out: when the
        const unsigned cap = total;         // count exceeds it the host falls back (AXB_ERR_STATE) and nothing is read
        total = *total_dev;
        if (total > cap) return;
    }
    for (unsigned s = blockIdx.x * blockDim.x + threadIdx.x; s < total; s += gridDim.x * blockDim.x) {
    const int4 me = tmp[s];
    const unsigned lo = off[me.x], hi = off[me.x + 1];
    unsigned pos = lo;
    for (unsigned q = lo; q < hi; ++q) {
        const int4 o = tmp[q];
        if (o.y < me.y || (o.y == me.y && (o.z < me.z || (o.z == me.z && o.w < me.w)))) ++pos;
        else if (o.y == me.y && o.z == me.z && o.w == me.w && q != s) atomicOr(&ctr->overflow, 1u << 5);
    }
    const auto w = out.row(pos, total, 4);
    w.put(0, mapped(map, me.x));
    w.put(1, mapped(map, me.y));
    w.put(2, mapped(map, me.z));
    w.put(3, mapped(map, me.w));
    }
}

template <class Out>
__global__ void __launch_bounds__(256) k_emit_tets(const int4 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                                   unsigned total, const uint32_t *__restrict__ total_dev,
                                                   const int64_t *__restrict__ map, Out out, Counters *ctr) {
    emit_tets_rows<Out>(tmp, off, total, total_dev, map, out, ctr);
}

// The four int64 lists in ONE launch (device-resident results, axb_compute_finish_into): layer blockIdx.y emits
// dimension y; the layers' tails overlap instead of following each other.
struct EmitAll {
    int n;
    const uint32_t *vkeep, *voff;
    const int2 *tmp1;
    const int4 *tmp2, *tmp3;
    const uint32_t *off1, *off2, *off3;
    unsigned cap[4];
    int64_t *out[4];
    Counters *ctr;
};
__global__ void __launch_bounds__(256) k_emit_all(EmitAll E) {
    if (blockIdx.y == 0) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E.n; i += gridDim.x * blockDim.x)
            if (E.vkeep[i] && E.voff[i] < E.cap[0]) E.out[0][E.voff[i]] = (int64_t)i;
    } else if (blockIdx.y == 1) {
        emit_edges_rows<PlainOut<int64_t>>(E.tmp1, E.off1, E.cap[1], E.off1 + E.n, nullptr, PlainOut<int64_t>{E.out[1]}, E.ctr);
    } else if (blockIdx.y == 2) {
        emit_tris_rows<PlainOut<int64_t>>(E.tmp2, E.off2, E.cap[2], E.off2 + E.n, nullptr, PlainOut<int64_t>{E.out[2]}, E.ctr);
    } else {
        emit_tets_rows<PlainOut<int64_t>>(E.tmp3, E.off3, E.cap[3], E.off3 + E.n, nullptr, PlainOut<int64_t>{E.out[3]}, E.ctr);
    }
}

template <class OutT>
__global__ void __launch_bounds__(256) k_emit_vertices(int n, const uint32_t *__restrict__ vkeep,
                                                       const uint32_t *__restrict__ voff,
                                                       const int64_t *__restrict__ map, OutT *__restrict__ out, unsigned cap) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (vkeep[i] && voff[i] < cap) out[voff[i]] = (OutT)mapped(map, i);
}

// ---- merge of canonical row lists from several slabs / chunks (reference pipeline.py:611-614):
// sorted union with duplicates removed.  Same owner-bucket scheme as above, plus a "first of its
// equals" mark so every distinct row is written once.
__device__ __forceinline__ int4 load_row4(const int64_t *__restrict__ rows, unsigned s, int k) {
    int4 r = make_int4(-1, -1, -1, -1);
    r.x = (int)rows[(size_t)s * k];
    if (k > 1) r.y = (int)rows[(size_t)s * k + 1];
    if (k > 2) r.z = (int)rows[(size_t)s * k + 2];
    if (k > 3) r.w = (int)rows[(size_t)s * k + 3];
    return r;
}

__device__ __forceinline__ bool row_less(const int4 &a, const int4 &b) {   // same owner (x)
    return a.y < b.y || (a.y == b.y && (a.z < b.z || (a.z == b.z && a.w < b.w)));
}
__device__ __forceinline__ bool row_equal(const int4 &a, const int4 &b) { return a.y == b.y && a.z == b.z && a.w == b.w; }

// (`base`: the rows' first column lies in [base, base + n_index) -- a rank that merges one index range of a sharded
// run sizes its bucket arrays for that range only)
__global__ void __launch_bounds__(256) k_merge_count(const int64_t *__restrict__ rows, unsigned m, int k, unsigned n_index,
                                                     int64_t base, uint32_t *__restrict__ cnt, Counters *ctr) {
    unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    const int64_t a = rows[(size_t)s * k] - base;
    if (a < 0 || a >= (int64_t)n_index) { atomicOr(&ctr->overflow, 1u << 6); return; }
    atomicAdd(cnt + a, 1u);
}

__global__ void __launch_bounds__(256) k_merge_scatter(const int64_t *__restrict__ rows, unsigned m, int k, unsigned n_index,
                                                       int64_t base, uint32_t *__restrict__ cnt, const uint32_t *__restrict__ off,
                                                       int4 *__restrict__ tmp) {
    unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    int4 r = load_row4(rows, s, k);
    const int64_t a = rows[(size_t)s * k] - base;
    if (a < 0 || a >= (int64_t)n_index) return;
    r.x = (int)a;                                    // bucket = owner relative to the range
    const unsigned slot = atomicSub(cnt + r.x, 1u) - 1u;
    tmp[off[r.x] + slot] = r;
}

__global__ void __launch_bounds__(256) k_merge_mark(const int4 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                                    unsigned m, uint32_t *__restrict__ ucnt, unsigned char *__restrict__ dup) {
    unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    const int4 me = tmp[s];
    if (me.x < 0) { dup[s] = 1; return; }
    const unsigned lo = off[me.x];
    bool d = false;
    for (unsigned q = lo; q < s && !d; ++q) d = row_equal(tmp[q], me);
    dup[s] = d ? 1 : 0;
    if (!d) atomicAdd(ucnt + me.x, 1u);
}

__global__ void __launch_bounds__(256) k_merge_emit(const int4 *__restrict__ tmp, const uint32_t *__restrict__ off,
                                                    const uint32_t *__restrict__ uoff, const unsigned char *__restrict__ dup,
                                                    unsigned m, int k, int64_t base, int64_t *__restrict__ out) {
    unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m || dup[s]) return;
    const int4 me = tmp[s];
    const unsigned lo = off[me.x], hi = off[me.x + 1];
    unsigned pos = uoff[me.x];
    for (unsigned q = lo; q < hi; ++q)
        if (!dup[q] && row_less(tmp[q], me)) ++pos;
    out[(size_t)pos * k] = (int64_t)me.x + base;
    if (k > 1) out[(size_t)pos * k + 1] = me.y;
    if (k > 2) out[(size_t)pos * k + 2] = me.z;
    if (k > 3) out[(size_t)pos * k + 3] = me.w;
}

}  // namespace axb
