// prune.cuh -- stage two: top-down pruning (reference pipeline.py:482-527).
//
// The reference computes, per level,  K_d = unique(faces(K_{d+1}) U free_d[AC2])
// with free_d = potential_d \ faces(K_{d+1}).  As sets that equals
// faces(K_{d+1}) U potential_d[AC2], so "free" is only a way to skip AC2 tests
// whose outcome cannot matter -- which is exactly how it is used here:
//   * every kept tetrahedron marks its 4 faces and 6 edges as kept,
//   * a potential triangle runs AC2 only if no kept tet marked it, and a kept
//     triangle marks its 3 edges,
//   * a potential edge runs AC2 only if nothing marked it; kept edges mark
//     their endpoints; unmarked viable vertices run AC2 at their own centre.
// Kept triangles are bits in the per-edge-row mask `trimask` (row = generator's
// partner slot i, bit = partner slot j > i), kept edges are `eflag` per
// potential edge, kept vertices `vflag` per rank.  The first time a simplex
// becomes kept, the counter of its owner (= minimum BALL INDEX vertex, which
// is the first column of its canonical row) is bumped, so the canonical
// output offsets are known without another pass.
// Ortho-centres are recomputed from the vertices instead of being stored:
// the solve is cheaper than a 32-byte round trip through HBM per simplex.
#pragma once

#include "common.cuh"
#include "predicates.cuh"

namespace axb {

struct PruneParams {
    GridView g;
    Tol tol;
    const Atom *atoms;
    const int *orig;
    const uint32_t *adj_off;
    const int *deg;
    const int *pe_u;
    const int *pe_v;
    const int4 *pt;
    const int4 *pq_r;
    const int *pq_l;
    uint32_t pt_cap, pq_cap, pe_cap;
    int W;                            // 64-bit words per trimask row
    unsigned long long *trimask;      // (n_pe, W)
    unsigned int *eflag;              // (n_pe)
    unsigned char *vflag;             // (n) by rank
    int4 *k3;                         // kept tets as ascending ball indices
    uint32_t *cnt1, *cnt2, *cnt3;     // per owner ball index
    uint32_t *vkeep;                  // per ball index, 0/1
    Counters *ctr;
    int biomolecule;
    int rank_lo, rank_hi;             // generators this call owns; rows of other generators only receive marks
    int own_only;                     // slab: count / list only the kept simplices whose generator is owned (every simplex
                                      // is then emitted by exactly one slab); otherwise a chunk also emits inherited faces
    uint32_t k3_cap;                  // capacity of k3
    int claim_tris, claim_edges;      // list entries per lane and work claim (k_prune_tris / k_prune_edges)
    // alpha sweep (sweep.cuh): the lists were built once at the largest alpha of the sweep.  Ortho-sizes and AC2
    // outcomes do not depend on alpha, so they were evaluated once for every listed simplex; what is left per alpha is
    // "potential at THIS alpha" (all edges flagged in sw_pf, sizes <= lim_a) and the inheritance marks.
    int sweep;
    const unsigned char *sw_pf;       // (n_pe) the edge passes the reach pre-filter and the size test at this alpha
    const double *sw_tsize;           // (n_pt) ortho-size of the triangle
    const int *sw_tvw;                // (n_pt) list position of its edge (v, w)
    const double *sw_qsize;           // (n_pq) ortho-size of the tet
    const double *sw_qtsize;          // (n_pq) ortho-size of its generating triangle (u, v, w)
    const int4 *sw_qe;                // (n_pq) list positions of its edges (v, w), (v, x), (w, x)
    const unsigned char *sw_ac2e, *sw_ac2t, *sw_ac2q;   // AC2 outcome per listed edge / triangle / tet
};

// slot of `target` in a generator's partner list; four independent loads per round, no early exit
// inside a round (the list has ~5-20 entries, so this is 2-5 memory round trips instead of up to 20)
__device__ __forceinline__ int find_partner(const int *__restrict__ pe_v, unsigned base, int d, int target) {
    int hit = -1;
    for (int q = 0; q < d && hit < 0; q += 4) {
        const int a0 = __ldg(pe_v + base + q);
        const int a1 = __ldg(pe_v + base + min(q + 1, d - 1));
        const int a2 = __ldg(pe_v + base + min(q + 2, d - 1));
        const int a3 = __ldg(pe_v + base + min(q + 3, d - 1));
        if (a3 == target) hit = min(q + 3, d - 1);
        if (a2 == target) hit = min(q + 2, d - 1);
        if (a1 == target) hit = min(q + 1, d - 1);
        if (a0 == target) hit = q;
    }
    return hit;
}

// The three look-ups a kept tet needs -- w and x in v's row, x in w's row -- as ONE loop: both rows are read four
// entries at a time in the same round (a warp issues in order: three look-ups one after the other were three to six
// dependent round trips, this is one or two).  Rows are duplicate-free, so a clamped re-read finds the same slot.
__device__ __forceinline__ void find_partners3(const int *__restrict__ pe_v, unsigned bv, int dv, int tw, int tx, unsigned bw,
                                               int dw, int tx2, int &iw, int &ix, int &jx) {
    iw = -1; ix = -1; jx = -1;
    const int dmax = max(dv, dw);
    for (int q = 0; q < dmax; q += 4) {
        int a[4], b[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k] = dv > 0 ? __ldg(pe_v + bv + min(q + k, dv - 1)) : -1;
            b[k] = dw > 0 ? __ldg(pe_v + bw + min(q + k, dw - 1)) : -1;
        }
#pragma unroll
        for (int k = 3; k >= 0; --k) {
            if (a[k] == tw) iw = min(q + k, dv - 1);
            if (a[k] == tx) ix = min(q + k, dv - 1);
            if (b[k] == tx2) jx = min(q + k, dw - 1);
        }
        const bool v_done = (iw >= 0 && ix >= 0) || q + 4 >= dv, w_done = jx >= 0 || q + 4 >= dw;
        if (v_done && w_done) break;
    }
}

#ifndef PRUNE_EARLY_MARKS
#define PRUNE_EARLY_MARKS 1      // triangles: the look-up's row base is requested before the solve
#endif
#ifndef PRUNE_EARLY_TETS
#define PRUNE_EARLY_TETS 0       // tets: the same (five more live values across the walk)
#endif
#ifndef PRUNE_MERGED_TETS
#define PRUNE_MERGED_TETS 1      // tets: the three look-ups as one loop (find_partners3)
#endif

// does this call emit the simplices generated by rank `gen`?
__device__ __forceinline__ bool emits(const PruneParams &P, int gen) {
    return !P.own_only || (gen >= P.rank_lo && gen < P.rank_hi);
}

__device__ __forceinline__ void mark_edge(const PruneParams &P, unsigned e, int owner, int gen) {
    unsigned old = atomicExch(P.eflag + e, 1u);
    if (!old && emits(P, gen)) atomicAdd(P.cnt1 + owner, 1u);
}

__device__ __forceinline__ void note_miss(const PruneParams &P) {
    atomicAdd(&P.ctr->lookup_miss, 1u);
    atomicOr(&P.ctr->overflow, 1u << 3);
}

__device__ __forceinline__ int min3(int a, int b, int c) { return min(a, min(b, c)); }

// AC2 of one simplex: the latency-tolerant walk when the dense cell table exists (rows = this thread's
// column of a [9][blockDim.x] shared table), the plain one for the sorted sparse grid
#ifndef AXB_AC2_MLP
#define AXB_AC2_MLP 1
#endif
__device__ __forceinline__ bool ac2_check(const PruneParams &P, double cx, double cy, double cz, double thr, int inc0,
                                          int inc1, int inc2, int inc3, int2 *rows, int stride) {
#if AXB_AC2_MLP
    if (P.g.cell_start) return ac2_pass_mlp(P.g, P.atoms, cx, cy, cz, thr, P.tol.r2max, inc0, inc1, inc2, inc3, rows, stride);
#endif
    return ac2_pass(P.g, P.atoms, cx, cy, cz, thr, P.tol.r2max, inc0, inc1, inc2, inc3);
}

// pipeline.py:496-497 (K3 = tets[AC2]) + inheritance of faces (pipeline.py:501, 509)
// NB: when a potential list overflowed its buffer (optimistic sizing in axb_compute) the tail of the
// buffer is garbage; every prune kernel then does nothing and the host re-runs with exact sizes.
__device__ __forceinline__ bool lists_overflowed(const PruneParams &P) {
    return P.ctr->n_pq > P.pq_cap || P.ctr->n_pt > P.pt_cap || P.ctr->n_pe > P.pe_cap;
}

#ifndef PRUNE_GRID
#define PRUNE_GRID 4        // blocks per SM launched = resident blocks (work is claimed dynamically)
#endif
#ifndef TETS_CLAIM_V
#define TETS_CLAIM_V 128
#endif
#ifndef TETS_MINB
#define TETS_MINB 3
#endif
#ifndef TETS_GRID
#define TETS_GRID 8         // blocks per SM of the static variant (TETS_MINB are resident at a time)
#endif
template <int DYN>
__global__ void __launch_bounds__(256, TETS_MINB) k_prune_tets(PruneParams P) {
    __shared__ int2 s_rows[9][256];
    if (lists_overflowed(P)) return;
    const unsigned n_pq = min(P.ctr->n_pq, P.pq_cap);
    // a warp claims 32 tets at a time from a global counter (dense regions make tets very unequal); the
    // next claim is issued before the current chunk is processed
    // DYN = 0: plain grid-stride loop (best while there are only a few tets per thread).
    // DYN = 1: a warp claims 128 tets at a time from a global counter -- dense regions make tets very
    // unequal -- and issues the next claim before it works on the current one.  Same-address atomics are
    // served at ~1 per ns, so claims must stay coarse (measured at 1M atoms, alpha 1.4: 32 per claim 1.47 ms,
    // 64 1.23 ms, 128 1.12 ms, 256 1.15 ms and worse in dense cores).
    constexpr unsigned CLAIM = TETS_CLAIM_V;
    const int lane = lane_id();
    unsigned chunk_n = 0;
    if (DYN && lane == 0) chunk_n = atomicAdd(&P.ctr->work_next[0], 1u);
    const unsigned stride = DYN ? 32u : gridDim.x * blockDim.x;
    for (;;) {
        unsigned e0, e1;
        if (DYN) {
            const unsigned chunk = __shfl_sync(FULL, chunk_n, 0);
            if ((unsigned long long)chunk * CLAIM >= n_pq) break;
            if (lane == 0) chunk_n = atomicAdd(&P.ctr->work_next[0], 1u);
            e0 = chunk * CLAIM + (unsigned)lane;
            e1 = min(chunk * CLAIM + CLAIM, n_pq);
        } else {
            e0 = blockIdx.x * blockDim.x + threadIdx.x;
            e1 = n_pq;
        }
      for (unsigned e = e0; e < e1; e += stride) {
        const int4 r = P.pq_r[e];
        if (r.w < P.rank_lo) continue;      // slab: no owned vertex (ranks ascend), the lower neighbour settles it
        const int l = P.pq_l[e];
        const int i = l & SLOT_MASK, j = (l >> SLOT_BITS) & SLOT_MASK, k = (l >> (2 * SLOT_BITS)) & SLOT_MASK;
        const int ou = __ldg(P.orig + r.x), ov = __ldg(P.orig + r.y), ow = __ldg(P.orig + r.z), ox = __ldg(P.orig + r.w);
#if PRUNE_EARLY_TETS
        // what the marks of a kept tet need is requested now: it arrives behind the solve and the walk
        const unsigned bu = __ldg(P.adj_off + r.x), bv = __ldg(P.adj_off + r.y), bw = __ldg(P.adj_off + r.z);
        const int dv = __ldg(P.deg + r.y), dw = __ldg(P.deg + r.z);
#endif
        if (P.sweep) {       // potential at this alpha (pipeline.py:447-478: six potential edges, both sizes) and AC2
            if (!P.sw_ac2q[e] || !(P.sw_qsize[e] <= P.tol.lim_a) || !(P.sw_qtsize[e] <= P.tol.lim_a)) continue;
            const unsigned b0 = __ldg(P.adj_off + r.x);
            const int4 qe = P.sw_qe[e];
            if (!(P.sw_pf[b0 + i] & P.sw_pf[b0 + j] & P.sw_pf[b0 + k] & P.sw_pf[qe.x] & P.sw_pf[qe.y] & P.sw_pf[qe.z])) continue;
        } else {
            const Atom au = load_atom(P.atoms, r.x), av = load_atom(P.atoms, r.y);
            const Atom aw = load_atom(P.atoms, r.z), ax = load_atom(P.atoms, r.w);
            const Ortho o = ortho_tet(ou, au, ov, av, ow, aw, ox, ax, P.tol.eps_sing);
#if PRUNE_EARLY_TETS
            if (dv > 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.pe_v + bv));     // the rows of the look-ups
            if (dw > 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.pe_v + bw));
#endif
            if (!ac2_check(P, o.cx, o.cy, o.cz, o.size - P.tol.eps_abs, r.x, r.y, r.z, r.w, &s_rows[0][threadIdx.x], 256)) continue;
        }
        int row[4] = {ou, ov, ow, ox};
#pragma unroll
        for (int a = 1; a < 4; ++a)
#pragma unroll
            for (int b = a; b > 0; --b)
                if (row[b - 1] > row[b]) { int t = row[b]; row[b] = row[b - 1]; row[b - 1] = t; }
        const bool own_u = emits(P, r.x), own_v = emits(P, r.y), own_w = emits(P, r.z);
        if (own_u) {
            const unsigned slot = atomicAdd(&P.ctr->n_k3, 1u);
            if (slot < P.k3_cap) P.k3[slot] = make_int4(row[0], row[1], row[2], row[3]);
            atomicAdd(P.cnt3 + row[0], 1u);
        }
        // Inheritance marks (pipeline.py:501, 509): 4 faces, 6 edges.  All lookups first, then all
        // atomics back to back (their round trips overlap), then the owner counters of what was new.
#if !PRUNE_EARLY_TETS
        const unsigned bu = __ldg(P.adj_off + r.x);
        const unsigned bv = __ldg(P.adj_off + r.y);
        const unsigned bw = __ldg(P.adj_off + r.z);
        const int dv = __ldg(P.deg + r.y), dw = __ldg(P.deg + r.z);
#endif
#if PRUNE_MERGED_TETS
        int iw, ix, jx;     // face (v, w, x) and edges (v, w), (v, x) live in v's rows, edge (w, x) in w's row
        find_partners3(P.pe_v, bv, dv, r.z, r.w, bw, dw, r.w, iw, ix, jx);
#else
        const int iw = find_partner(P.pe_v, bv, dv, r.z);       // face (v, w, x) and edges (v, w), (v, x) live in v's rows
        const int ix = find_partner(P.pe_v, bv, dv, r.w);
        const int jx = find_partner(P.pe_v, bw, dw, r.w);       // edge (w, x) in w's row
#endif
        const unsigned long long bj = 1ull << (j & 63), bk = 1ull << (k & 63);
        const size_t W = (size_t)P.W;
        const unsigned long long t0 = atomicOr(P.trimask + (size_t)(bu + i) * W + (j >> 6), bj);
        const unsigned long long t1 = atomicOr(P.trimask + (size_t)(bu + i) * W + (k >> 6), bk);
        const unsigned long long t2 = atomicOr(P.trimask + (size_t)(bu + j) * W + (k >> 6), bk);
        unsigned long long t3 = ~0ull;
        const unsigned long long bx = 1ull << (ix & 63);
        if (iw >= 0 && ix >= 0) t3 = atomicOr(P.trimask + (size_t)(bv + iw) * W + (ix >> 6), bx);
        const unsigned e0 = atomicExch(P.eflag + bu + i, 1u);
        const unsigned e1 = atomicExch(P.eflag + bu + j, 1u);
        const unsigned e2 = atomicExch(P.eflag + bu + k, 1u);
        const unsigned e3 = iw >= 0 ? atomicExch(P.eflag + bv + iw, 1u) : 1u;
        const unsigned e4 = ix >= 0 ? atomicExch(P.eflag + bv + ix, 1u) : 1u;
        const unsigned e5 = jx >= 0 ? atomicExch(P.eflag + bw + jx, 1u) : 1u;
        // (a face is generated by its minimum-rank vertex: u, or v for the face opposite u, or w for the edge (w, x))
        if (own_u) {
            if (!(t0 & bj)) atomicAdd(P.cnt2 + min3(ou, ov, ow), 1u);
            if (!(t1 & bk)) atomicAdd(P.cnt2 + min3(ou, ov, ox), 1u);
            if (!(t2 & bk)) atomicAdd(P.cnt2 + min3(ou, ow, ox), 1u);
            if (!e0) atomicAdd(P.cnt1 + min(ou, ov), 1u);
            if (!e1) atomicAdd(P.cnt1 + min(ou, ow), 1u);
            if (!e2) atomicAdd(P.cnt1 + min(ou, ox), 1u);
        }
        if (own_v) {
            if (iw >= 0 && ix >= 0 && !(t3 & bx)) atomicAdd(P.cnt2 + min3(ov, ow, ox), 1u);
            if (!e3) atomicAdd(P.cnt1 + min(ov, ow), 1u);
            if (!e4) atomicAdd(P.cnt1 + min(ov, ox), 1u);
        }
        if (!e5 && own_w) atomicAdd(P.cnt1 + min(ow, ox), 1u);
        if (iw < 0 || ix < 0) { note_miss(P); if (iw < 0) note_miss(P); if (ix < 0) note_miss(P); }
        if (jx < 0) note_miss(P);
      }
        if (!DYN) break;
    }
}

#ifndef PRUNE_THREADS_V
#define PRUNE_THREADS_V 256
#endif
constexpr int PRUNE_THREADS = PRUNE_THREADS_V;
#ifndef PRUNE_MINB
#define PRUNE_MINB 4      // <= 64 registers: measured best (occupancy beats the few spilled values)
#endif

// Warp-autonomous work compaction for the two kernels below: most potential triangles / edges are
// already kept by inheritance, so a warp claims chunks of the list from a global counter, pushes the
// FREE entries onto its own shared-memory stack and runs the expensive part (ortho solve + AC2) whenever
// 32 are waiting -- packed lanes, no block barriers, and dense regions do not leave other warps idle.
constexpr int PRUNE_WARPS = PRUNE_THREADS / 32;
// the triangle kernel wants a few more registers than four blocks of 256 threads leave (64: 36 B of spills); seven warps
// per block are 28 warps per SM at 72 registers (0.241 -> 0.229 ms at 1M atoms); the edge kernel is better off at 64
#ifndef TRIS_THREADS_V
#define TRIS_THREADS_V 224
#endif
constexpr int TRIS_THREADS = TRIS_THREADS_V;
constexpr int TRIS_WARPS = TRIS_THREADS / 32;
// List entries per lane and claim: coarse claims keep a warp inside one neighbourhood (L1) and spare the shared
// counter, fine ones keep every warp busy when the list is short.  Measured on B200 (tools/gpu_autotune.sh):
// 1M atoms 4 / 6 (triangles / edges) beat 2 by 11 / 20 %, 50k atoms want 1; larger than 8 loses to tail imbalance.
#ifndef PRUNE_CLAIM_TRIS
#define PRUNE_CLAIM_TRIS 4
#endif
#ifndef PRUNE_CLAIM_EDGES
#define PRUNE_CLAIM_EDGES 6
#endif
// host side: the claim for a list of `entries` worked on by `warps` resident warps (at least ~4 claims per warp)
inline int prune_claim(unsigned long long entries, unsigned warps, int large) {
    const unsigned long long per = entries / ((unsigned long long)warps * 32ull * 4ull);
    return (int)(per < 1 ? 1 : per > (unsigned long long)large ? (unsigned long long)large : per);
}
#ifndef PRUNE_SCAN_U
#define PRUNE_SCAN_U 4
#endif
constexpr int PRUNE_STACK = 32 + 32 * PRUNE_SCAN_U;   // free entries parked per warp (processed as soon as 32 are waiting;
                                                      // a scan step adds up to 32 * PRUNE_SCAN_U)

// pipeline.py:502-505: AC2 for the triangles no kept tet inherited
__global__ void __launch_bounds__(TRIS_THREADS, PRUNE_MINB) k_prune_tris(PruneParams P) {
    __shared__ unsigned s_stack[TRIS_WARPS][PRUNE_STACK];
    __shared__ int2 s_rows[9][TRIS_THREADS];
    if (lists_overflowed(P)) return;
    const unsigned n_pt = min(P.ctr->n_pt, P.pt_cap);
    const int lane = lane_id();
    unsigned *stack = s_stack[threadIdx.x >> 5];
    int sn = 0;                                       // warp-uniform stack fill

    auto settle = [&](unsigned e) {                   // one free triangle per lane
        const int4 r = P.pt[e];
        const int i = r.w & 0xffff, j = (r.w >> 16) & 0x7fff;
        const unsigned bu = __ldg(P.adj_off + r.x);
        const int ou = __ldg(P.orig + r.x), ov = __ldg(P.orig + r.y), ow = __ldg(P.orig + r.z);
#if PRUNE_EARLY_MARKS
        const unsigned bv = __ldg(P.adj_off + r.y);          // for the marks: requested now, arrives behind the solve
        const int dv = __ldg(P.deg + r.y);
#endif
        if (P.sweep) {       // potential at this alpha (pipeline.py:398-420: three potential edges, own size) and AC2
            if (!P.sw_ac2t[e] || !(P.sw_tsize[e] <= P.tol.lim_a)) return;
            if (!(P.sw_pf[bu + i] & P.sw_pf[bu + j] & P.sw_pf[P.sw_tvw[e]])) return;
        } else {
            const Atom au = load_atom(P.atoms, r.x), av = load_atom(P.atoms, r.y), aw = load_atom(P.atoms, r.z);
            const Ortho o = ortho_tri(ou, au, ov, av, ow, aw, P.tol.eps_sing);
#if PRUNE_EARLY_MARKS
            if (dv > 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.pe_v + bv));     // the row of the look-up
#endif
            if (!ac2_check(P, o.cx, o.cy, o.cz, o.size - P.tol.eps_abs, r.x, r.y, r.z, -1, &s_rows[0][threadIdx.x], TRIS_THREADS)) return;
        }
        // kept: mark the triangle and its three edges.  The lookup first, then all four atomics back to back (their
        // round trips overlap), then the owner counters of what was new (no return value needed: fire and forget)
#if PRUNE_EARLY_MARKS
        const int iw = find_partner(P.pe_v, bv, dv, r.z);
#else
        const unsigned bv = __ldg(P.adj_off + r.y);
        const int iw = find_partner(P.pe_v, bv, __ldg(P.deg + r.y), r.z);
#endif
        const unsigned long long bit = 1ull << (j & 63);
        const unsigned long long t0 = atomicOr(P.trimask + (size_t)(bu + i) * P.W + (j >> 6), bit);
        const unsigned e0 = atomicExch(P.eflag + bu + i, 1u);
        const unsigned e1 = atomicExch(P.eflag + bu + j, 1u);
        const unsigned e2 = iw >= 0 ? atomicExch(P.eflag + bv + iw, 1u) : 1u;
        if (emits(P, r.x)) {
            if (!(t0 & bit)) atomicAdd(P.cnt2 + min3(ou, ov, ow), 1u);
            if (!e0) atomicAdd(P.cnt1 + min(ou, ov), 1u);
            if (!e1) atomicAdd(P.cnt1 + min(ou, ow), 1u);
        }
        if (!e2 && emits(P, r.y)) atomicAdd(P.cnt1 + min(ov, ow), 1u);
        if (iw < 0) note_miss(P);
    };

    // fill the stack from claimed chunks until 32 free entries wait (or the list is exhausted), then settle
    // up to 32 of them -- ONE call site of the expensive part keeps the register allocation tight
    const int claim = P.claim_tris;
    const unsigned span = 32u * (unsigned)claim;
    unsigned chunk_n = 0, chunk = 0;
    int b = claim;                                    // sub-step inside the current chunk (claim = need a new one)
    bool exhausted = false;
    if (lane == 0) chunk_n = atomicAdd(&P.ctr->work_next[1], 1u);
    for (;;) {
        while (sn < 32 && !exhausted) {
            if (b == claim) {
                chunk = __shfl_sync(FULL, chunk_n, 0);
                if ((unsigned long long)chunk * span >= n_pt) { exhausted = true; break; }
                if (lane == 0) chunk_n = atomicAdd(&P.ctr->work_next[1], 1u);
                b = 0;
            }
            // PRUNE_SCAN_U sub-steps of the claim at once, level by level (list entry -> row base -> mask word): a warp
            // issues in order, so one entry per iteration made every iteration wait for three dependent round trips
            constexpr int U = PRUNE_SCAN_U;
            const unsigned ebase = chunk * span + (unsigned)(b * 32 + lane);
            const int nsub = min(U, claim - b);
            b += nsub;
            int4 r[U];
            bool c[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const unsigned e = ebase + 32u * k;
                r[k] = make_int4(0, 0, 0, -1);
                if (k < nsub && e < n_pt) r[k] = P.pt[e];
            }
            unsigned bu[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                // bit 31: already known to be dominated (cull mode); slab: a triangle below every owned ball is the
                // lower neighbour's
                c[k] = r[k].w >= 0 && r[k].z >= P.rank_lo;
                bu[k] = c[k] ? __ldg(P.adj_off + r[k].x) : 0u;
            }
            unsigned long long w[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = (r[k].w >> 16) & 0x7fff;
                w[k] = c[k] ? P.trimask[(size_t)(bu[k] + (r[k].w & 0xffff)) * P.W + (j >> 6)] : ~0ull;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = (r[k].w >> 16) & 0x7fff;
                const bool f = c[k] && !((w[k] >> (j & 63)) & 1ull);     // not inherited from a kept tet
                const unsigned m = __ballot_sync(FULL, f);
                if (f) stack[sn + __popc(m & lanemask_lt())] = ebase + 32u * k;
                sn += __popc(m);
            }
            __syncwarp();
        }
        if (sn == 0) break;
        const int take = min(sn, 32);
        sn -= take;
        const unsigned mine = stack[sn + min(lane, take - 1)];
        __syncwarp();
        if (lane < take) settle(mine);
    }
}

// pipeline.py:510-513: AC2 for the edges nothing inherited; kept edges mark their endpoints
__global__ void __launch_bounds__(PRUNE_THREADS, PRUNE_MINB) k_prune_edges(PruneParams P) {
    __shared__ unsigned s_stack[PRUNE_WARPS][PRUNE_STACK];
    __shared__ int2 s_rows[9][PRUNE_THREADS];
    if (lists_overflowed(P)) return;
    const unsigned n_pe = min(P.ctr->n_pe, P.pe_cap);
    const int lane = lane_id();
    unsigned *stack = s_stack[threadIdx.x >> 5];
    int sn = 0;

    auto settle = [&](unsigned e) {
        const int u = __ldg(P.pe_u + e), v = __ldg(P.pe_v + e);
        const int ou = __ldg(P.orig + u), ov = __ldg(P.orig + v);
        bool keep;
        if (P.sweep) {
            keep = P.sw_pf[e] && P.sw_ac2e[e];
        } else {
            const Atom au = load_atom(P.atoms, u), av = load_atom(P.atoms, v);
            const Ortho o = ortho_edge(ou, au, ov, av, P.tol.eps_sing);
            keep = ac2_check(P, o.cx, o.cy, o.cz, o.size - P.tol.eps_abs, u, v, -1, -1, &s_rows[0][threadIdx.x], PRUNE_THREADS);
        }
        if (keep) {
            mark_edge(P, e, min(ou, ov), u);
            P.vflag[u] = 1;
            P.vflag[v] = 1;
        }
    };

    const int claim = P.claim_edges;
    const unsigned span = 32u * (unsigned)claim;
    unsigned chunk_n = 0, chunk = 0;
    int b = claim;
    bool exhausted = false;
    if (lane == 0) chunk_n = atomicAdd(&P.ctr->work_next[2], 1u);
    for (;;) {
        while (sn < 32 && !exhausted) {
            if (b == claim) {
                chunk = __shfl_sync(FULL, chunk_n, 0);
                if ((unsigned long long)chunk * span >= n_pe) { exhausted = true; break; }
                if (lane == 0) chunk_n = atomicAdd(&P.ctr->work_next[2], 1u);
                b = 0;
            }
            // PRUNE_SCAN_U sub-steps of the claim at once (see k_prune_tris)
            constexpr int U = PRUNE_SCAN_U;
            const unsigned ebase = chunk * span + (unsigned)(b * 32 + lane);
            const int nsub = min(U, claim - b);
            b += nsub;
            int eu[U], ev[U];
            unsigned ef[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const unsigned e = ebase + 32u * k;
                const bool valid = k < nsub && e < n_pe;
                eu[k] = valid ? __ldg(P.pe_u + e) : -1;
                ev[k] = valid ? __ldg(P.pe_v + e) : -1;
                ef[k] = valid ? P.eflag[e] : 0u;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                bool is_free = false;
                if (eu[k] >= 0) {
                    if (ef[k] != 0u) {                            // inherited: its endpoints are kept
                        P.vflag[eu[k]] = 1;
                        P.vflag[ev[k]] = 1;
                    } else {
                        // slab: an edge below every owned ball or generated by the upper halo is a neighbour's business
                        is_free = eu[k] < P.rank_hi && ev[k] >= P.rank_lo;
                    }
                }
                const unsigned m = __ballot_sync(FULL, is_free);
                if (is_free) stack[sn + __popc(m & lanemask_lt())] = ebase + 32u * k;
                sn += __popc(m);
            }
            __syncwarp();
        }
        if (sn == 0) break;
        const int take = min(sn, 32);
        sn -= take;
        const unsigned mine = stack[sn + min(lane, take - 1)];
        __syncwarp();
        if (lane < take) settle(mine);
    }
}

// pipeline.py:517-525: vertices.  Endpoints of kept edges are kept wherever they live; the own
// domination check only runs for the balls this call owns (ranks [rank_lo, rank_hi) = vertex_ids).
__global__ void __launch_bounds__(256) k_prune_vertices(PruneParams P, int rank_lo, int rank_hi) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.g.n) return;
    bool kept = P.vflag[t] != 0;
    if (!kept && t >= rank_lo && t < rank_hi) {
        kept = P.biomolecule != 0;
        if (!kept) {
            const Atom a = load_atom(P.atoms, t);
            if (-a.r2 <= P.tol.lim_a)                                  // pipeline.py:520
                kept = ac2_pass(P.g, P.atoms, a.x, a.y, a.z, -a.r2 - P.tol.eps_abs, P.tol.r2max, t, -1, -1, -1);
        }
    }
    P.vkeep[__ldg(P.orig + t)] = (kept && emits(P, t)) ? 1u : 0u;
}

}  // namespace axb
