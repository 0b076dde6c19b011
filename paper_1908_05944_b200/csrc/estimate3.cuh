// estimate3.cuh -- potential triangles and tetrahedra, warp-autonomous tiles
// (reference pipeline.py:373-479).
//
// Every WARP owns a tile of up to 16 consecutive generators and its own slice of shared memory;
// nothing but __syncwarp separates the phases, so the warps of a block (and the blocks of an SM)
// drift apart and hide each other's fp64 dependency chains (a block-per-tile predecessor spent a
// quarter of its stall cycles at block barriers):
//   A  stage the partner atoms of the tile (generators and partners share ONE index space in
//      shared memory, so "sort the vertices by ball index" is a sort of four small integers
//      followed by loads in sorted order -- no 32-byte records are swapped in registers)
//   B  lane = partner slot i, round r pairs it with slot i + r of the same generator: reach
//      pre-filter (pipeline.py:398-401), passing pairs queued with ballot/popc; the queue is solved
//      a full warp at a time: ortho2 -> bit matrix M ("pair is a potential edge", pipeline.py:412-415),
//      ortho3 -> bit matrix T (potential triangle, pipeline.py:417-420)
//   C  warp scan over the T rows numbers the tile's triangles (one contiguous run of the global
//      list per tile); every partner slot expands its own row and counts its tet candidates
//      M[i] & M[j] & (bits > j)  (pipeline.py:447, 455-466: both new edges must be potential)
//   D  warp scan numbers the candidates; one lane per candidate runs ortho4 (pipeline.py:475-478);
//      kept tets are compacted with ballot/popc and ONE global atomic per warp round.
// Cull mode: see dominated_by_partner3.
#pragma once

#include "common.cuh"
#include "estimate.cuh"
#include "predicates.cuh"

namespace axb {

#ifndef T3_WARPS_V
#define T3_WARPS_V 4
#endif
constexpr int T3_WARPS = T3_WARPS_V;      // warps per block (each one is independent)
// Tile shapes (template parameter SHAPE): the light shape packs lanes best when a generator has ~11 partner
// pairs (alpha = 0); the heavy shape shrinks the tile (6 generators, ~6 KB of shared memory per warp) so that 32 warps fit
// an SM at 64 registers -- faster once generators have 40+ pairs (alpha = 1.4, dense cores; 1M atoms, alpha 1.4: 5 / 6 / 7 /
// 8 blocks per SM = 2.31 / 2.19 / 2.12 / 2.04 ms), slower at alpha = 0.
enum { T3_LIGHT = 0, T3_HEAVY = 1, T3_SMALL = 2 };   // T3_SMALL: the light algorithm at 16 warps per SM, no spilled values
                                                     // (few tiles per warp: nothing hides a slower tile)
constexpr int T3_WQCAP = 288;             // reach-passing pairs queued (solved as soon as 256 are waiting)

// heavy tile shape (tuning knobs, tools/gpu_autotune.sh: 6 generators / 160 triangles per round beat 8 / 112 by 5 % at
// 1M atoms, alpha 1.4 -- 8 generators with ~10 partners each overflow the 64 slots and split the tile -- and by 2 % in
// dense cores; 4 generators or more slots per tile lose)
#ifndef T3H_GENS
#define T3H_GENS 6
#endif
#ifndef T3H_SCAP
#define T3H_SCAP 64
#endif
#ifndef T3H_TCAP
#define T3H_TCAP 160
#endif
#ifndef T3H_MINB
#define T3H_MINB 8
#endif

// light tile shape.  The kernel's time goes with 1 / resident warps up to 16 per SM (4, 8, 12, 16 warps: 1.55, 0.82, 0.58,
// 0.46 ms at 1M atoms, alpha 0) and flattens beyond: with the single solve site (see phase B) 20 warps at 96 registers are
// the optimum (0.384 ms; 16 warps 0.415, 24 warps at 80 registers 0.46: the flat pair path spills there); at most 9.4 KB
// of shared memory per warp (96 partner slots, 160 triangles per round).  Smaller tiles for more warps lose (12
// generators at 24 warps 0.457 ms, 8 at 32 warps 0.489 ms).
#ifndef T3L_GENS
#define T3L_GENS 16
#endif
#ifndef T3L_SCAP
#define T3L_SCAP 96
#endif
#ifndef T3L_TCAP
#define T3L_TCAP 160
#endif
#ifndef T3L_MINB
#define T3L_MINB 5
#endif
#ifndef T3L_PTAB
#define T3L_PTAB 640
#endif
// cull mode bit 1 (triangles flagged as dominated by a partner, AXB_CULL=2|3) needs a third bit matrix per warp; it
// never paid, so it is compiled out unless asked for
#ifndef T3_SPEC3
#define T3_SPEC3 1
#endif
#ifndef T3_CULL2
#define T3_CULL2 2
#endif
#ifndef T3_PAIR2
#define T3_PAIR2 1
#endif
#ifndef T3_STAGE_MLP
#define T3_STAGE_MLP 1
#endif
#ifndef T3_CULL_TRIS
#define T3_CULL_TRIS 0
#endif

template <int W, int SHAPE>
struct T3Cfg {
    static constexpr int GENS = (W == 1 && SHAPE == T3_HEAVY) ? T3H_GENS : (W == 1 && SHAPE == T3_LIGHT) ? T3L_GENS : 16;   // generators per warp tile (<= 16)
    static constexpr int SCAP = W == 1 ? (SHAPE == T3_HEAVY ? T3H_SCAP : SHAPE == T3_SMALL ? 128 : T3L_SCAP) : 256;   // partner slots per sub-pass (>= 64 * W)
    static constexpr int TCAP = W == 1 ? (SHAPE == T3_HEAVY ? T3H_TCAP : SHAPE == T3_SMALL ? 224 : T3L_TCAP) : 512;  // triangles per round
    static constexpr int MINB = W == 1 ? (SHAPE == T3_HEAVY ? T3H_MINB : SHAPE == T3_SMALL ? 4 : T3L_MINB) : 1;        // resident blocks per SM the registers must allow
    static constexpr int NA = SCAP + GENS;              // atom index space: partner slots, then the tile's generators
    static constexpr bool FLAT = W == 1 && SHAPE != T3_HEAVY;   // flattened pair enumeration (pays while degrees are small)
    static constexpr int PTAB = FLAT ? (SHAPE == T3_SMALL ? 1024 : T3L_PTAB) : 32;   // partner pairs of a sub-pass covered by the stamped pair table
};

template <int W, int SHAPE>
struct T3Warp {
    using C = T3Cfg<W, SHAPE>;
    double ax[C::NA], ay[C::NA], az[C::NA], ar2[C::NA];
    double sreach[C::SCAP];
    unsigned long long M[C::SCAP * W];
    unsigned long long T[C::SCAP * W];
#if T3_CULL_TRIS
    unsigned long long D[C::SCAP * W];         // potential triangles already known to be dominated (cull mode bit 1)
#endif
    int aorig[C::NA];
    int srank[C::SCAP];
    int rowpre[C::SCAP + 1];
    int gdeg[C::GENS];
    unsigned gadj[C::GENS];
    int sp[C::GENS + 1];                       // slot prefix over the whole tile
    unsigned short tl[C::TCAP];                // triangles of the round: slot i | slot j << 8 (filled in phase B while they fit)
    union {
        unsigned short wq[T3_WQCAP];           // phase B: queue of reach-passing pairs (slot i | slot j << 8)
        int cpre[C::TCAP + 1];                 // phases C, D: tet candidates per triangle, scanned
    } u;
    unsigned char sgen[C::SCAP], sli[C::SCAP];
    unsigned char ptab[C::PTAB];               // pair number -> first slot of the pair (phase B, flattened enumeration)
};

// largest idx in [0, n) with pre[idx] <= v (pre = exclusive prefix, pre[0] = 0)
__device__ __forceinline__ int owner_of(const int *pre, int n, int v) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (pre[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

// position of the nth set bit of a W-word row (-1 if there are fewer)
template <int W>
__device__ __forceinline__ int nth_bit_multi(const unsigned long long *row, int nth) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
        unsigned long long m = row[w];
        int c = __popcll(m);
        if (nth < c) return 64 * w + nth_set_bit(m, nth);
        nth -= c;
    }
    return -1;
}

// exclusive scan of a[0..n) in place by one warp; a[n] = total; returns the total
__device__ __forceinline__ int warp_scan_excl(int *a, int n) {
    const int lane = lane_id();
    int carry = 0;
    for (int b = 0; b < n; b += 32) {
        const int i = b + lane;
        const int v = i < n ? a[i] : 0;
        const int incl = warp_incl_scan(v);
        if (i < n) a[i] = carry + incl - v;
        carry += __shfl_sync(FULL, incl, 31);
    }
    if (lane == 0) a[n] = carry;
    __syncwarp();
    return carry;
}

template <class SW>
__device__ __forceinline__ Atom atom_at(const SW &S, int a) {
    Atom p;
    p.x = S.ax[a]; p.y = S.ay[a]; p.z = S.az[a]; p.r2 = S.ar2[a];
    return p;
}

// bit j of a row of 64-bit words, as a native 32-bit shared-memory atomic (little endian: word j >> 5)
__device__ __forceinline__ void set_bit(unsigned long long *row, int j) {
    atomicOr(reinterpret_cast<unsigned int *>(row) + (j >> 5), 1u << (j & 31));
}

__device__ __forceinline__ void cswap_idx(int &oa, int &ia, int &ob, int &ib) {
    if (oa > ob) { int t = oa; oa = ob; ob = t; t = ia; ia = ib; ib = t; }
}

// ortho solves on atoms named by their shared-memory index: sort (ball index, slot) pairs, then load in order
template <class SW>
__device__ __forceinline__ Ortho ortho_edge_s(const SW &S, int a, int b, double eps_sing) {
    int oa = S.aorig[a], ob = S.aorig[b];
    cswap_idx(oa, a, ob, b);
    return ortho2(atom_at(S, a), atom_at(S, b), eps_sing);
}

template <class SW>
__device__ __forceinline__ Ortho ortho_tri_s(const SW &S, int a, int b, int c, double eps_sing) {
    int oa = S.aorig[a], ob = S.aorig[b], oc = S.aorig[c];
    cswap_idx(oa, a, ob, b);
    cswap_idx(ob, b, oc, c);
    cswap_idx(oa, a, ob, b);
    const Atom p[3] = {atom_at(S, a), atom_at(S, b), atom_at(S, c)};
    return orthoN<3>(p, eps_sing);
}

template <class SW>
__device__ __forceinline__ Ortho ortho_tet_s(const SW &S, int a, int b, int c, int d, double eps_sing) {
    int oa = S.aorig[a], ob = S.aorig[b], oc = S.aorig[c], od = S.aorig[d];
    cswap_idx(oa, a, ob, b);
    cswap_idx(oc, c, od, d);
    cswap_idx(oa, a, oc, c);
    cswap_idx(ob, b, od, d);
    cswap_idx(ob, b, oc, c);
    const Atom p[4] = {atom_at(S, a), atom_at(S, b), atom_at(S, c), atom_at(S, d)};
    return orthoN<4>(p, eps_sing);
}

// Cull mode (the one-call path; the standalone stage API needs the complete potential lists and
// switches it off): a simplex whose ortho-centre is dominated by another partner of its generator
// fails the domination check of the pruning stage for certain -- a dominating ball is closer than
// one cell side to the centre (pipeline.py:288-289), so it is one of the 27-cell candidates, and the
// power distance below is evaluated exactly like pipeline.py:308-309.  The partners are already in
// shared memory, so most dominated simplices are settled here and never reach the AC2 kernels.
template <class SW>
__device__ __forceinline__ bool dominated_by_partner3(const SW &S, int sb, int se, int s0, int s1, int s2,
                                                      double cx, double cy, double cz, double thr) {
#if T3_CULL2
    // T3_CULL2 partners per iteration (independent fp64 chains: a thread issues in order; the simplex' own slots are
    // masked afterwards -- they sit at the simplex' size, above the threshold up to rounding)
    constexpr int K = T3_CULL2;
    for (int s = sb; s < se; s += K) {
        double dp[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int t = min(s + k, se - 1);
            const double ax = S.ax[t] - cx, ay = S.ay[t] - cy, az = S.az[t] - cz;
            dp[k] = ((ax * ax + ay * ay) + az * az) - S.ar2[t];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int t = min(s + k, se - 1);
            if (dp[k] < thr && !(t == s0 || t == s1 || t == s2)) return true;
        }
    }
    return false;
#else
    for (int s = sb; s < se; ++s) {
        if (s == s0 || s == s1 || s == s2) continue;
        const double ddx = S.ax[s] - cx, ddy = S.ay[s] - cy, ddz = S.az[s] - cz;
        const double dp = ((ddx * ddx + ddy * ddy) + ddz * ddz) - S.ar2[s];
        if (dp < thr) return true;
    }
    return false;
#endif
}

// ordinal of triangle (s, sj) among its generator's triangles in (i, j) order, from the listed triangles of the tile
// (error path only: the ordinal goes into the key that picks the first singular simplex, pipeline.py:475-477)
__device__ __noinline__ unsigned listed_tri_ordinal(const unsigned short *tl, const unsigned char *sgen, int ntri, int s, int sj) {
    const int g = sgen[s];
    unsigned before = 0;
    for (int y = 0; y < ntri; ++y) {
        const int a = tl[y] & 0xff, b = tl[y] >> 8;
        if (sgen[a] == g && (a < s || (a == s && b < sj))) ++before;
    }
    return before;
}

template <int W, int SHAPE>
__global__ void __launch_bounds__(T3_WARPS * 32, (T3Cfg<W, SHAPE>::MINB)) k_tri_tet3(EstParams P, int rank_lo, int rank_hi) {
    using C = T3Cfg<W, SHAPE>;
    constexpr int T3_GENS = C::GENS;
    constexpr int PCAP = 64 * W;
    constexpr int SCAP = C::SCAP, TCAP = C::TCAP;
    extern __shared__ __align__(16) unsigned char s_raw3[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    T3Warp<W, SHAPE> &S = reinterpret_cast<T3Warp<W, SHAPE> *>(s_raw3)[warp];
    const int ntiles = (rank_hi - rank_lo + T3_GENS - 1) / T3_GENS;

    // Tiles are claimed from a global counter (dense regions make tiles very unequal); the claim for the
    // NEXT tile is issued before the current one is processed, so its round trip is hidden.
    int tile_n = 0;
    if (lane == 0) tile_n = (int)atomicAdd(&P.ctr->tile_next, 1u);
    for (;;) {
        const int tile = __shfl_sync(FULL, tile_n, 0);
        if (tile >= ntiles) break;
        if (lane == 0) tile_n = (int)atomicAdd(&P.ctr->tile_next, 1u);
        const int t0 = rank_lo + tile * T3_GENS;
        const int ng_all = min(T3_GENS, rank_hi - t0);
        __syncwarp();                                       // previous tile fully consumed
        {   // generators of the tile: atom index SCAP + g
            int d = 0;
            if (lane < ng_all) {
                d = __ldg(P.deg + t0 + lane);
                if (d < 2 || d > PCAP) d = 0;               // no partner pair: nothing to do; too many for a tile: heavy.cuh
                S.gadj[lane] = __ldg(P.adj_off + t0 + lane);
                // slab, lower halo: only simplices that reach an owned ball matter (partners ascend in rank)
                if (d && t0 + lane < P.own_lo && __ldg(P.pe_v + S.gadj[lane] + d - 1) < P.own_lo) d = 0;
                const Atom a = load_atom(P.atoms, t0 + lane);
                S.ax[SCAP + lane] = a.x; S.ay[SCAP + lane] = a.y; S.az[SCAP + lane] = a.z; S.ar2[SCAP + lane] = a.r2;
                S.aorig[SCAP + lane] = __ldg(P.orig + t0 + lane);
            }
            if (lane < T3_GENS) S.gdeg[lane] = d;
            const int incl = warp_incl_scan(d);
            if (lane < T3_GENS) S.sp[lane + 1] = incl;
            if (lane == 0) S.sp[0] = 0;
        }
        __syncwarp();
        int g0 = 0;
        while (g0 < ng_all) {
            // ---- sub-pass [g0, g1): as many generators as fit the slot budget (normally the whole tile)
            const int base = S.sp[g0];
            int g1;
            {
                const bool in = lane >= g0 && lane < ng_all && S.sp[lane + 1] - base <= SCAP;
                g1 = g0 + __popc(__ballot_sync(FULL, in));  // slot counts are monotone: the set is a prefix
            }
            const int nslots = S.sp[g1] - base;
            int npairs_any = 0;
            if (lane >= g0 && lane < g1) npairs_any = S.gdeg[lane];
            if (__ballot_sync(FULL, npairs_any > 0) != 0u) {
                // ---- A: stage the partner atoms (ascending rank inside a generator = pipeline.py:362-370)
#if T3_STAGE_MLP
                if constexpr (W == 1) {
                    // A warp issues in order: with one slot per loop iteration the second slot's rank is only requested
                    // after the first slot's record has arrived (its store to shared memory waits for it).  So: the
                    // ranks of ALL the lane's slots first, then all records, then the stores -- two round trips per
                    // sub-pass instead of two per 32 slots.
                    constexpr int SL = (SCAP + 31) / 32;
                    int srk[SL], sg[SL];
#pragma unroll
                    for (int k = 0; k < SL; ++k) {
                        const int s = lane + 32 * k;
                        sg[k] = -1;
                        srk[k] = 0;
                        if (s < nslots) {
                            int g = g0;                     // last generator with sp[g] - base <= s
#pragma unroll
                            for (int step = 8; step > 0; step >>= 1)
                                if (g + step < g1 && S.sp[g + step] - base <= s) g += step;
                            sg[k] = g;
                            srk[k] = __ldg(P.pe_v + S.gadj[g] + (s - (S.sp[g] - base)));
                        }
                    }
                    Atom sa[SL];
                    double sr[SL];
                    int so[SL];
#pragma unroll
                    for (int k = 0; k < SL; ++k) {
                        sa[k].x = sa[k].y = sa[k].z = sa[k].r2 = 0.0; sr[k] = 0.0; so[k] = 0;
                        if (sg[k] >= 0) {
                            sa[k] = load_atom(P.atoms, srk[k]);
                            sr[k] = __ldg(P.reach + srk[k]);
                            so[k] = __ldg(P.orig + srk[k]);
                        }
                    }
#pragma unroll
                    for (int k = 0; k < SL; ++k) {
                        const int s = lane + 32 * k;
                        if (sg[k] >= 0) {
                            S.ax[s] = sa[k].x; S.ay[s] = sa[k].y; S.az[s] = sa[k].z; S.ar2[s] = sa[k].r2;
                            S.sreach[s] = sr[k];
                            S.aorig[s] = so[k];
                            S.srank[s] = srk[k];
                            S.sgen[s] = (unsigned char)sg[k];
                            S.sli[s] = (unsigned char)(s - (S.sp[sg[k]] - base));
                            S.M[s] = 0ull; S.T[s] = 0ull;
#if T3_CULL_TRIS
                            S.D[s] = 0ull;
#endif
                        }
                    }
                } else
#endif
                for (int s = lane; s < nslots; s += 32) {
                    int g = g0;                             // last generator with sp[g] - base <= s
#pragma unroll
                    for (int step = 8; step > 0; step >>= 1)
                        if (g + step < g1 && S.sp[g + step] - base <= s) g += step;
                    const int li = s - (S.sp[g] - base);
                    const int rk = __ldg(P.pe_v + S.gadj[g] + li);
                    const Atom a = load_atom(P.atoms, rk);
                    S.ax[s] = a.x; S.ay[s] = a.y; S.az[s] = a.z; S.ar2[s] = a.r2;
                    S.sreach[s] = __ldg(P.reach + rk);
                    S.aorig[s] = __ldg(P.orig + rk);
                    S.srank[s] = rk;
                    S.sgen[s] = (unsigned char)g;
                    S.sli[s] = (unsigned char)li;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        S.M[s * W + w] = 0ull; S.T[s * W + w] = 0ull;
#if T3_CULL_TRIS
                        S.D[s * W + w] = 0ull;
#endif
                    }
                }
                __syncwarp();
                // ---- B: partner pairs.  Lane = partner slot i; round r pairs it with slot i + r of the same
                // generator (np.triu_indices order is irrelevant here: results are bits).
                int nt;                                                   // potential triangles of the sub-pass (warp-uniform)
                bool listed;                                              // ... and all of them are in S.tl, in (i, j) order
                {
                    unsigned short *wq = S.u.wq;
                    int qn = 0;                                           // warp-uniform queue fill
                    nt = 0;
                    listed = false;
                    auto solve_queue = [&](int count) {                    // dense ortho2 + ortho3 over wq[0..count)
                        for (int x0 = 0; x0 < count; x0 += 32) {
                            const int x = x0 + lane;
                            bool tri = false;
                            unsigned short pr = 0;
                            if (x < count) {
                                pr = wq[x];
                                const int si = (int)(pr & 0xffu), sj = (int)(pr >> 8);
                                const int g = S.sgen[si];
                                const int i = S.sli[si], j = S.sli[sj];
                                const int t = t0 + g;
                                const int d = S.gdeg[g];
                                const unsigned q = (unsigned)(i * (2 * d - i - 1) / 2 + (j - i - 1));   // triu ordinal
                                const Ortho e2 = ortho_edge_s(S, si, sj, P.tol.eps_sing);                // pipeline.py:412-414
#if T3_SPEC3
                                // (solved beside the edge, not behind it: nearly every pre-filtered pair is a potential edge,
                                // and two independent fp64 chains fill the issue slots one leaves empty; its result and its
                                // singular flag only count if the pair passes, as in the reference)
                                const Ortho e3 = ortho_tri_s(S, SCAP + g, si, sj, P.tol.eps_sing);       // pipeline.py:417-419
#endif
                                if (e2.singular) record_singular(P, make_err_key(ST_VW, t, q), S.aorig[si], S.aorig[sj], -1, -1, 2);
                                if (e2.size <= P.tol.lim_a) {                                            // pipeline.py:415
                                    set_bit(&S.M[si * W], j);
                                    set_bit(&S.M[sj * W], i);
#if !T3_SPEC3
                                    const Ortho e3 = ortho_tri_s(S, SCAP + g, si, sj, P.tol.eps_sing);   // pipeline.py:417-419
#endif
                                    if (e3.singular)
                                        record_singular(P, make_err_key(ST_TRI, t, q), S.aorig[SCAP + g], S.aorig[si], S.aorig[sj], -1, 3);
                                    if (e3.size <= P.tol.lim_a) {                                        // pipeline.py:420
                                        set_bit(&S.T[si * W], j);
                                        tri = true;
#if T3_CULL_TRIS
                                        if (P.cull & 2) {
                                            const int sb = S.sp[g] - base;
                                            if (dominated_by_partner3(S, sb, sb + d, si, sj, -1, e3.cx, e3.cy, e3.cz, e3.size - P.tol.eps_abs))
                                                set_bit(&S.D[si * W], j);
                                        }
#endif
                                    }
                                }
                            }
                            // the triangle goes straight into the round's list (the queue is in (i, j) order, so is the
                            // list) while the tile's triangles fit one round -- they nearly always do; the T rows are
                            // only expanded otherwise
                            const unsigned tm = __ballot_sync(FULL, tri);
                            if (tm) {
                                if (listed && nt + __popc(tm) <= TCAP) {
                                    if (tri) S.tl[nt + __popc(tm & lanemask_lt())] = pr;
                                } else {
                                    listed = false;
                                }
                                nt += __popc(tm);
                            }
                        }
                        __syncwarp();
                    };
                    // Pair numbering: slot i owns the pairs (i, i + 1 .. i + more_i); an exclusive scan of `more` over the
                    // slots numbers them.  When the pair table covers the sub-pass (SCAP < 256 slots, so one byte names a
                    // slot) every slot stamps its range and the pre-filter runs over the FLATTENED pairs with packed
                    // lanes; the slot-by-offset loop below keeps only half its lanes busy and runs to the largest
                    // degree of each 32-slot group.  Light tile shape only: with 40+ pairs per generator the second
                    // set of shared loads per pair costs more than the idle lanes (measured: -7 % at alpha = 0, +5..16 %
                    // at alpha = 1.4 and in dense cores).
                    int npairs = 0x7fffffff;
                    if constexpr (C::FLAT) {
                        for (int s = lane; s < nslots; s += 32) S.rowpre[s] = S.gdeg[S.sgen[s]] - 1 - (int)S.sli[s];
                        __syncwarp();
                        npairs = warp_scan_excl(S.rowpre, nslots);
                    }
                    // The enumeration is RESUMABLE and the queue is solved at ONE call site: five inlined copies of the two
                    // ortho solves made the kernel 4,500 instructions long, and with every warp in a phase of its own
                    // instruction fetch was the third largest stall reason (ncu r2g: no_instruction 1.6 per issue).
                    const bool flat = C::FLAT && npairs <= C::PTAB;
                    if (flat) {
                        listed = true;                      // pairs are queued in (i, j) order: so are the triangles
                        for (int s = lane; s < nslots; s += 32) {
                            const int pb = S.rowpre[s], pe = S.rowpre[s + 1];
                            for (int p = pb; p < pe; ++p) S.ptab[p] = (unsigned char)s;
                        }
                        __syncwarp();
                    }
                    int p0 = 0;                             // flat: next pair number
                    int s0 = -32, r = 1, rounds = 0;        // slot by offset: group of 32 slots, round inside the group
                    bool done = false;
                    while (!done) {
                        if (flat) {
#if T3_PAIR2
                            // two pairs per lane and iteration (the table look-ups of both are in flight together)
                            while (p0 < npairs && qn < 32 * 7) {
                                const int pa = p0 + lane, pb = pa + 32;
                                p0 += 64;
                                bool passa = false, passb = false;
                                int sia = 0, sja = 0, sib = 0, sjb = 0;
                                if (pa < npairs) sia = S.ptab[pa];
                                if (pb < npairs) sib = S.ptab[pb];
                                if (pa < npairs) sja = sia + 1 + (pa - S.rowpre[sia]);
                                if (pb < npairs) sjb = sib + 1 + (pb - S.rowpre[sib]);
                                if (pa < npairs) passa = reach_pair(atom_at(S, sia), S.sreach[sia], atom_at(S, sja), S.sreach[sja]);   // pipeline.py:398-401
                                if (pb < npairs) passb = reach_pair(atom_at(S, sib), S.sreach[sib], atom_at(S, sjb), S.sreach[sjb]);
                                const unsigned ma = __ballot_sync(FULL, passa), mb = __ballot_sync(FULL, passb);
                                if (passa) wq[qn + __popc(ma & lanemask_lt())] = (unsigned short)(sia | (sja << 8));
                                qn += __popc(ma);
                                if (passb) wq[qn + __popc(mb & lanemask_lt())] = (unsigned short)(sib | (sjb << 8));
                                qn += __popc(mb);
                            }
                            done = p0 >= npairs;
#else
                            while (p0 < npairs && qn < 32 * 8) {
                                const int p = p0 + lane;
                                p0 += 32;
                                bool pass = false;
                                int si = 0, sj = 0;
                                if (p < npairs) {
                                    si = S.ptab[p];
                                    sj = si + 1 + (p - S.rowpre[si]);
                                    pass = reach_pair(atom_at(S, si), S.sreach[si], atom_at(S, sj), S.sreach[sj]);   // pipeline.py:398-401
                                }
                                const unsigned m = __ballot_sync(FULL, pass);
                                if (pass) wq[qn + __popc(m & lanemask_lt())] = (unsigned short)(si | (sj << 8));
                                qn += __popc(m);
                            }
                            done = p0 >= npairs;
#endif
                        } else {
                            // lane = slot i of the group, round r pairs it with slot i + r (its record is re-read after a
                            // solve instead of being kept alive across it)
                            int more = 0;
                            Atom av;
                            double rv = 0.0;
                            av.x = av.y = av.z = av.r2 = 0.0;
                            const int si = s0 + lane;
                            if (s0 >= 0 && si < nslots) {
                                more = S.gdeg[S.sgen[si]] - 1 - (int)S.sli[si];   // partners after slot i in its generator
                                av = atom_at(S, si);
                                rv = S.sreach[si];
                            }
                            while (qn < 32 * 8) {
                                if (r > rounds) {           // next group
                                    s0 += 32;
                                    if (s0 >= nslots) { done = true; break; }
                                    break;                  // (re-enter with the new group's records)
                                }
                                bool pass = false;
                                const int sj = si + r;
                                if (r <= more) pass = reach_pair(av, rv, atom_at(S, sj), S.sreach[sj]);   // pipeline.py:398-401
                                ++r;
                                const unsigned m = __ballot_sync(FULL, pass);
                                if (pass) wq[qn + __popc(m & lanemask_lt())] = (unsigned short)(si | (sj << 8));
                                qn += __popc(m);
                            }
                            if (!done && r > rounds && qn < 32 * 8) {
                                // the new group: how many rounds it needs
                                int mr = 0;
                                const int sn = s0 + lane;
                                if (sn < nslots) mr = S.gdeg[S.sgen[sn]] - 1 - (int)S.sli[sn];
#pragma unroll
                                for (int o = 16; o > 0; o >>= 1) mr = max(mr, __shfl_xor_sync(FULL, mr, o));
                                rounds = mr;
                                r = 1;
                                continue;                   // nothing to solve yet
                            }
                        }
                        __syncwarp();
                        solve_queue(qn);
                        qn = 0;
                    }
                }
                // ---- C: triangle list of the tile
                if (!listed) {
                    for (int s = lane; s < nslots; s += 32) {
                        int c = 0;
#pragma unroll
                        for (int w = 0; w < W; ++w) c += __popcll(S.T[s * W + w]);
                        S.rowpre[s] = c;
                    }
                    __syncwarp();
                    warp_scan_excl(S.rowpre, nslots);
                }
                const int ntri = nt;
                // one contiguous run of the global triangle list per tile: the prune kernel that reads it
                // then works on one neighbourhood at a time (L1 locality)
                unsigned pt_base = 0;
                if (lane == 0 && ntri > 0) pt_base = atomicAdd(&P.ctr->n_pt, (unsigned)ntri);
                pt_base = __shfl_sync(FULL, pt_base, 0);
                for (int tc0 = 0; tc0 < ntri; tc0 += TCAP) {
                    const int ntc = min(TCAP, ntri - tc0);
                    if (listed) {
                        // lane = triangle: its tet candidates are the partners above j adjacent (in M) to both i and j:
                        // rank[x] > rank_hi (pipeline.py:447)
                        for (int x = lane; x < ntc; x += 32) {
                            const int srow = S.tl[x] & 0xff, sj = S.tl[x] >> 8;
                            const int j = S.sli[sj];
                            int cnt = 0;
#pragma unroll
                            for (int w2 = 0; w2 < W; ++w2) {
                                unsigned long long m = S.M[srow * W + w2] & S.M[sj * W + w2];
                                const int lowbit = j + 1 - 64 * w2;
                                if (lowbit >= 64) m = 0ull;
                                else if (lowbit > 0) m &= ~0ull << lowbit;
                                cnt += __popcll(m);
                            }
                            S.u.cpre[x] = cnt;
                            const unsigned pos = pt_base + (unsigned)x;
#if T3_CULL_TRIS
                            const int dom = (int)((S.D[srow * W + (j >> 6)] >> (j & 63)) & 1ull);
#else
                            const int dom = 0;
#endif
                            if (pos < P.pt_cap)
                                P.pt[pos] = make_int4(t0 + (int)S.sgen[srow], S.srank[srow], S.srank[sj],
                                                      (int)S.sli[srow] | (j << 16) | (dom << 31));
                        }
                    } else
                    // every partner slot expands its own triangles (bits of its T row) into the round's list
                    for (int srow = lane; srow < nslots; srow += 32) {
                        int tt = S.rowpre[srow];
                        if (tt >= tc0 + ntc || S.rowpre[srow + 1] <= tc0) continue;
                        const int g = S.sgen[srow];
                        const int sg = S.sp[g] - base;
#pragma unroll
                        for (int w = 0; w < W; ++w) {
                            unsigned long long bits = S.T[srow * W + w];
                            while (bits) {
                                const int j = 64 * w + __ffsll((long long)bits) - 1;
                                bits &= bits - 1;
                                const int x = tt - tc0;
                                ++tt;
                                if (x < 0 || x >= ntc) continue;
                                const int sj = sg + j;
                                S.tl[x] = (unsigned short)(srow | (sj << 8));
                                // partners above j adjacent (in M) to both: rank[x] > rank_hi (pipeline.py:447)
                                int cnt = 0;
#pragma unroll
                                for (int w2 = 0; w2 < W; ++w2) {
                                    unsigned long long m = S.M[srow * W + w2] & S.M[sj * W + w2];
                                    const int lowbit = j + 1 - 64 * w2;
                                    if (lowbit >= 64) m = 0ull;
                                    else if (lowbit > 0) m &= ~0ull << lowbit;
                                    cnt += __popcll(m);
                                }
                                S.u.cpre[x] = cnt;
                                const unsigned pos = pt_base + (unsigned)(tc0 + x);
#if T3_CULL_TRIS
                                const int dom = (int)((S.D[srow * W + (j >> 6)] >> (j & 63)) & 1ull);
#else
                                const int dom = 0;
#endif
                                if (pos < P.pt_cap)
                                    P.pt[pos] = make_int4(t0 + g, S.srank[srow], S.srank[sj],
                                                          (int)S.sli[srow] | (j << 16) | (dom << 31));
                            }
                        }
                    }
                    __syncwarp();
                    const int ncand = warp_scan_excl(S.u.cpre, ntc);
                    // ---- D: dense over tet candidates (pipeline.py:447-479)
                    for (int c0 = 0; c0 < ncand; c0 += 32) {
                        const int c = c0 + lane;
                        bool keep = false;
                        int4 er = make_int4(0, 0, 0, 0);
                        int el = 0;
                        if (c < ncand) {
                            const int x = owner_of(S.u.cpre, ntc, c);
                            const int s = S.tl[x] & 0xff, sj = S.tl[x] >> 8;
                            const int j = S.sli[sj];
                            unsigned long long cm[W];
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                unsigned long long m = S.M[s * W + w] & S.M[sj * W + w];
                                const int lowbit = j + 1 - 64 * w;
                                if (lowbit >= 64) m = 0ull;
                                else if (lowbit > 0) m &= ~0ull << lowbit;
                                cm[w] = m;
                            }
                            const int k = nth_bit_multi<W>(cm, c - S.u.cpre[x]);
                            const int g = S.sgen[s];
                            const int sb = S.sp[g] - base;
                            const int sk = sb + k;
                            const int t = t0 + g;
                            const Ortho e4 = ortho_tet_s(S, SCAP + g, s, sj, sk, P.tol.eps_sing);        // pipeline.py:475-477
                            if (e4.singular) {
                                const unsigned tri_ord = listed ? listed_tri_ordinal(S.tl, S.sgen, ntc, s, sj)
                                                                : (unsigned)(tc0 + x - S.rowpre[sb]);    // ordinal among u's triangles
                                record_singular(P, make_err_key(ST_TET, t, tet_ordinal(tri_ord, k)), S.aorig[SCAP + g],
                                                S.aorig[s], S.aorig[sj], S.aorig[sk], 4);
                            }
                            keep = e4.size <= P.tol.lim_a;                                               // pipeline.py:478
                            if (keep && (P.cull & 1) &&
                                dominated_by_partner3(S, sb, sb + S.gdeg[g], s, sj, sk, e4.cx, e4.cy, e4.cz, e4.size - P.tol.eps_abs))
                                keep = false;        // AC2 would fail at this partner (it lies in the 27-cell block): never kept
                            er = make_int4(t, S.srank[s], S.srank[sj], S.srank[sk]);
                            el = pack_slots((int)S.sli[s], j, k);
                        }
                        const unsigned m = __ballot_sync(FULL, keep);
                        if (m) {
                            unsigned pq_base = 0;
                            if (lane == 0) pq_base = atomicAdd(&P.ctr->n_pq, (unsigned)__popc(m));
                            pq_base = __shfl_sync(FULL, pq_base, 0);
                            if (keep) {
                                const unsigned pos = pq_base + (unsigned)__popc(m & lanemask_lt());
                                if (pos < P.pq_cap) { P.pq_r[pos] = er; P.pq_l[pos] = el; }
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
            g0 = g1;
        }
    }
}

}  // namespace axb
