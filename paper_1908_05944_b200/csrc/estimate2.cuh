// estimate2.cuh -- potential triangles and tetrahedra, block-per-tile version
// (reference pipeline.py:373-479).
//
// The warp-per-generator kernel of estimate.cuh kept only ~9 of 32 lanes busy
// (a generator has ~11 partner pairs, ~4 triangles, ~1 tet candidate).  Here a
// block of 256 threads takes a TILE of up to 128 consecutive generators, stages
// all their partner atoms in shared memory once, and runs every phase over the
// tile's FLATTENED work list so lanes stay packed:
//   B1  all partner pairs of the tile (np.triu_indices order inside a generator):
//       reach pre-filter, passing pairs appended to a shared list
//   B2  dense over the passing pairs: ortho2 (is the pair a potential edge? ->
//       bit matrix M), then ortho3 (potential triangle -> bit matrix T)
//   C   prefix over T rows -> the tile's triangle list; each triangle is written
//       to the global list and its tet candidates M[i]&M[j]&(bits > j) counted
//   D   prefix over candidate counts; dense over candidates: ortho4, size test,
//       kept tets written to the global list
// Output slots are claimed with one global atomic per warp and 32 items.
#pragma once

#include "common.cuh"
#include "estimate.cuh"
#include "predicates.cuh"

namespace axb {

#ifndef T2_THREADS_V
#define T2_THREADS_V 128
#endif
#ifndef T2_GENS_V
#define T2_GENS_V 64
#endif
#ifndef T2_MINB
#define T2_MINB 4
#endif
constexpr int T2_THREADS = T2_THREADS_V;
constexpr int T2_WARPS = T2_THREADS / 32;
constexpr int T2_GENS = T2_GENS_V;       // generators per tile (multiple of 32)
constexpr int T2_GPL = T2_GENS / 32;     // generators per lane in the tile prefix
constexpr int T2_SCAP = 8 * T2_GENS;     // partner slots per sub-pass (>= 64 * W so one generator always fits)
constexpr int T2_TCAP = 24 * T2_GENS;    // triangles per round
constexpr int T2_WQCAP = 288;            // reach-passing pairs queued per warp (solved as soon as 256 are waiting)
static_assert(T2_GENS % 32 == 0 && T2_GENS <= T2_THREADS && T2_SCAP >= 256, "tile shape");

template <int W>
struct T2Smem {
    double sx[T2_SCAP], sy[T2_SCAP], sz[T2_SCAP], sr2[T2_SCAP], sreach[T2_SCAP];
    double gx[T2_GENS], gy[T2_GENS], gz[T2_GENS], gr2[T2_GENS];
    unsigned long long M[T2_SCAP * W];
    unsigned long long T[T2_SCAP * W];
    unsigned long long D[T2_SCAP * W];         // potential triangles already known to be dominated (cull mode)
    int sorig[T2_SCAP], srank[T2_SCAP];
    int rowpre[T2_SCAP + 1];
    int gorig[T2_GENS], gdeg[T2_GENS];
    unsigned gadj[T2_GENS];
    int sp[T2_GENS + 1];           // slot prefix of the sub-pass
    int pp[T2_GENS + 1];           // pair prefix of the sub-pass
    union {
        unsigned wq[T2_WARPS][T2_WQCAP];       // phase B: per-warp queue of reach-passing pairs (slot i | slot j << 16)
        struct {
            unsigned short tri_si[T2_TCAP], tri_sj[T2_TCAP];
            int cpre[T2_TCAP + 1];
        } t;
    } u;
    unsigned char sgen[T2_SCAP], sli[T2_SCAP];
    int wtot[T2_WARPS + 1];
    int qoff[T2_WARPS];
    unsigned pt_base, pq_base;
    int npass;
    int g1;
    int fits;
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

// in-place exclusive scan of a[0..n) by the whole block; returns the total (also stored in a[n])
__device__ __forceinline__ int block_scan_excl(int *a, int n, int *wtot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + T2_THREADS - 1) / T2_THREADS;
    const int b = min(tid * per, n), e = min(b + per, n);
    int sum = 0;
    for (int i = b; i < e; ++i) sum += a[i];
    const int incl = warp_incl_scan(sum);
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int v = lane < T2_WARPS ? wtot[lane] : 0;
        int iv = warp_incl_scan(v);
        if (lane < T2_WARPS) wtot[lane] = iv - v;
        if (lane == T2_WARPS - 1) wtot[T2_WARPS] = iv;
    }
    __syncthreads();
    int off = wtot[warp] + incl - sum;
    for (int i = b; i < e; ++i) { int t = a[i]; a[i] = off; off += t; }
    const int total = wtot[T2_WARPS];
    if (tid == 0) a[n] = total;
    __syncthreads();
    return total;
}

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

// Cull mode (the one-call path; the standalone stage API needs the complete potential lists and
// switches it off): a simplex whose ortho-centre is dominated by another partner of its generator
// fails the domination check of the pruning stage for certain -- a dominating ball is closer than
// one cell side to the centre (pipeline.py:288-289), so it is one of the 27-cell candidates, and the
// power distance below is evaluated exactly like pipeline.py:308-309.  The partners are already in
// shared memory, so most dominated simplices are settled here and never reach the AC2 kernels.
template <int W>
__device__ __forceinline__ bool dominated_by_partner(const T2Smem<W> &S, int g, int g0, int s0, int s1, int s2,
                                                     double cx, double cy, double cz, double thr) {
    const int sb = S.sp[g], se = sb + S.gdeg[g0 + g];
    for (int s = sb; s < se; ++s) {
        if (s == s0 || s == s1 || s == s2) continue;
        const double ddx = S.sx[s] - cx, ddy = S.sy[s] - cy, ddz = S.sz[s] - cz;
        const double dp = ((ddx * ddx + ddy * ddy) + ddz * ddz) - S.sr2[s];
        if (dp < thr) return true;
    }
    return false;
}

template <int W>
__global__ void __launch_bounds__(T2_THREADS, T2_MINB) k_tri_tet2(EstParams P, int rank_lo, int rank_hi) {
    constexpr int PCAP = 64 * W;
    extern __shared__ __align__(16) unsigned char s_raw2[];
    T2Smem<W> &S = *reinterpret_cast<T2Smem<W> *>(s_raw2);
    const int tid = threadIdx.x, lane = tid & 31;
    const int ntiles = (rank_hi - rank_lo + T2_GENS - 1) / T2_GENS;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int t0 = rank_lo + tile * T2_GENS;
        const int ng_all = min(T2_GENS, rank_hi - t0);
        __syncthreads();                                    // previous tile fully consumed
        if (tid < T2_GENS) {
            int d = 0;
            if (tid < ng_all) {
                d = min(__ldg(P.deg + t0 + tid), PCAP);
                if (d < 2) d = 0;                           // no partner pair, nothing to do
                S.gadj[tid] = __ldg(P.adj_off + t0 + tid);
                const Atom a = load_atom(P.atoms, t0 + tid);
                S.gx[tid] = a.x; S.gy[tid] = a.y; S.gz[tid] = a.z; S.gr2[tid] = a.r2;
                S.gorig[tid] = __ldg(P.orig + t0 + tid);
            }
            S.gdeg[tid] = d;
        }
        __syncthreads();
        // slot / pair prefixes of the whole window (warp 0, T2_GPL generators per lane)
        if (tid < 32) {
            int d[T2_GPL], ls = 0, lp = 0;
#pragma unroll
            for (int k = 0; k < T2_GPL; ++k) { d[k] = S.gdeg[T2_GPL * tid + k]; ls += d[k]; lp += d[k] * (d[k] - 1) / 2; }
            const int is = warp_incl_scan(ls), ip = warp_incl_scan(lp);
            int es = is - ls, ep = ip - lp;
#pragma unroll
            for (int k = 0; k < T2_GPL; ++k) {
                S.sp[T2_GPL * tid + k] = es; S.pp[T2_GPL * tid + k] = ep;
                es += d[k]; ep += d[k] * (d[k] - 1) / 2;
            }
            if (tid == 31) { S.sp[T2_GENS] = es; S.pp[T2_GENS] = ep; S.fits = es <= T2_SCAP; }
        }
        __syncthreads();
        const bool fits = S.fits;
        int g0 = 0;
        while (g0 < ng_all) {
            // ---- sub-pass [g0, g1): the whole window when it fits the slot budget (the common case),
            // otherwise as many generators as fit, found by one thread
            if (!fits) {
                if (tid == 0) {
                    int slots = 0, pairs = 0, g = g0;
                    S.sp[0] = 0; S.pp[0] = 0;
                    while (g < ng_all && slots + S.gdeg[g] <= T2_SCAP) {
                        const int d = S.gdeg[g];
                        slots += d;
                        pairs += d * (d - 1) / 2;
                        ++g;
                        S.sp[g - g0] = slots;
                        S.pp[g - g0] = pairs;
                    }
                    S.g1 = g;
                }
                __syncthreads();
            } else if (tid == 0) {
                S.g1 = ng_all;
            }
            if (fits) __syncthreads();
            const int g1 = S.g1;
            const int ng = g1 - g0;
            const int nslots = S.sp[ng];
            const int npairs = S.pp[ng];
            if (npairs > 0) {
                // ---- A: stage the partner atoms (ascending rank inside a generator = pipeline.py:362-370)
                for (int s = tid; s < nslots; s += T2_THREADS) {
                    const int g = owner_of(S.sp, ng, s);
                    const int li = s - S.sp[g];
                    const int rk = __ldg(P.pe_v + S.gadj[g0 + g] + li);
                    const Atom a = load_atom(P.atoms, rk);
                    S.sx[s] = a.x; S.sy[s] = a.y; S.sz[s] = a.z; S.sr2[s] = a.r2;
                    S.sreach[s] = __ldg(P.reach + rk);
                    S.sorig[s] = __ldg(P.orig + rk);
                    S.srank[s] = rk;
                    S.sgen[s] = (unsigned char)g;
                    S.sli[s] = (unsigned char)li;
#pragma unroll
                    for (int w = 0; w < W; ++w) { S.M[s * W + w] = 0ull; S.T[s * W + w] = 0ull; S.D[s * W + w] = 0ull; }
                }
                __syncthreads();
                // ---- B: partner pairs, warp-autonomous.  Lane = partner slot i; round r pairs it with slot
                // i + r of the same generator (np.triu_indices order is irrelevant here: results are bits).
                // B1 queues the pairs that pass the reach pre-filter (pipeline.py:398-401) with a ballot;
                // B2 solves a full warp of queued pairs at a time, so the ortho code runs with packed lanes.
                {
                    const int warp = tid >> 5;
                    unsigned *wq = S.u.wq[warp];
                    int qn = 0;                                           // warp-uniform queue fill
                    auto solve_queue = [&](int count) {                    // dense ortho2 + ortho3 over wq[0..count)
                        for (int x0 = 0; x0 < count; x0 += 32) {
                            const int x = x0 + lane;
                            if (x < count) {
                                const unsigned pr = wq[x];
                                const int si = (int)(pr & 0xffffu), sj = (int)(pr >> 16);
                                const int g = S.sgen[si];
                                const int i = S.sli[si], j = S.sli[sj];
                                Atom av, aw;
                                av.x = S.sx[si]; av.y = S.sy[si]; av.z = S.sz[si]; av.r2 = S.sr2[si];
                                aw.x = S.sx[sj]; aw.y = S.sy[sj]; aw.z = S.sz[sj]; aw.r2 = S.sr2[sj];
                                const int ov = S.sorig[si], ow = S.sorig[sj];
                                const int t = t0 + g0 + g;
                                const int d = S.gdeg[g0 + g];
                                const unsigned q = (unsigned)(i * (2 * d - i - 1) / 2 + (j - i - 1));   // triu ordinal
                                const Ortho e2 = ortho_edge(ov, av, ow, aw, P.tol.eps_sing);             // pipeline.py:412-414
                                if (e2.singular) record_singular(P, make_err_key(ST_VW, t, q), ov, ow, -1, -1, 2);
                                if (e2.size <= P.tol.lim_a) {                                            // pipeline.py:415
                                    atomicOr(&S.M[si * W + (j >> 6)], 1ull << (j & 63));
                                    atomicOr(&S.M[sj * W + (i >> 6)], 1ull << (i & 63));
                                    Atom au;
                                    au.x = S.gx[g0 + g]; au.y = S.gy[g0 + g]; au.z = S.gz[g0 + g]; au.r2 = S.gr2[g0 + g];
                                    const int ou = S.gorig[g0 + g];
                                    const Ortho e3 = ortho_tri(ou, au, ov, av, ow, aw, P.tol.eps_sing);  // pipeline.py:417-419
                                    if (e3.singular) record_singular(P, make_err_key(ST_TRI, t, q), ou, ov, ow, -1, 3);
                                    if (e3.size <= P.tol.lim_a) {                                        // pipeline.py:420
                                        atomicOr(&S.T[si * W + (j >> 6)], 1ull << (j & 63));
                                        if ((P.cull & 2) && dominated_by_partner(S, g, g0, si, sj, -1, e3.cx, e3.cy, e3.cz,
                                                                           e3.size - P.tol.eps_abs))
                                            atomicOr(&S.D[si * W + (j >> 6)], 1ull << (j & 63));
                                    }
                                }
                            }
                        }
                        __syncwarp();
                    };
                    for (int s0 = warp * 32; s0 < nslots; s0 += T2_THREADS) {
                        const int si = s0 + lane;
                        int more = 0, sbase = 0;
                        Atom av;
                        double rv = 0.0;
                        av.x = av.y = av.z = av.r2 = 0.0;
                        if (si < nslots) {
                            const int g = S.sgen[si];
                            more = S.gdeg[g0 + g] - 1 - (int)S.sli[si];   // partners after slot i in its generator
                            sbase = si;
                            av.x = S.sx[si]; av.y = S.sy[si]; av.z = S.sz[si]; av.r2 = S.sr2[si];
                            rv = S.sreach[si];
                        }
                        int rounds = more;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(FULL, rounds, o));
                        for (int r = 1; r <= rounds; ++r) {
                            bool pass = false;
                            const int sj = sbase + r;
                            if (r <= more) {
                                Atom aw;
                                aw.x = S.sx[sj]; aw.y = S.sy[sj]; aw.z = S.sz[sj]; aw.r2 = S.sr2[sj];
                                pass = reach_pair(av, rv, aw, S.sreach[sj]);
                            }
                            const unsigned m = __ballot_sync(FULL, pass);
                            if (m) {
                                if (qn + 32 > T2_WQCAP) { __syncwarp(); solve_queue(qn); qn = 0; }
                                if (pass) wq[qn + __popc(m & lanemask_lt())] = (unsigned)si | ((unsigned)sj << 16);
                                qn += __popc(m);
                                __syncwarp();
                                if (qn >= 32 * 8) { solve_queue(qn); qn = 0; }
                            }
                        }
                    }
                    __syncwarp();
                    solve_queue(qn);
                }
                __syncthreads();
                // ---- C: triangle list of the tile
                for (int s = tid; s < nslots; s += T2_THREADS) {
                    int c = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) c += __popcll(S.T[s * W + w]);
                    S.rowpre[s] = c;
                }
                __syncthreads();
                const int ntri = block_scan_excl(S.rowpre, nslots, S.wtot);
                // one contiguous run of the global triangle list per tile: the prune kernel that reads it
                // then works on one neighbourhood at a time (L1 locality)
                if (tid == 0 && ntri > 0) S.pt_base = atomicAdd(&P.ctr->n_pt, (unsigned)ntri);
                __syncthreads();
                for (int tc0 = 0; tc0 < ntri; tc0 += T2_TCAP) {
                    const int ntc = min(T2_TCAP, ntri - tc0);
                    // every partner slot expands its own triangles (bits of its T row) into the round's list
                    for (int srow = tid; srow < nslots; srow += T2_THREADS) {
                        int tt = S.rowpre[srow];
                        if (tt >= tc0 + ntc || S.rowpre[srow + 1] <= tc0) continue;
                        const int g = S.sgen[srow];
#pragma unroll
                        for (int w = 0; w < W; ++w) {
                            unsigned long long bits = S.T[srow * W + w];
                            while (bits) {
                                const int j = 64 * w + __ffsll((long long)bits) - 1;
                                bits &= bits - 1;
                                const int x = tt - tc0;
                                ++tt;
                                if (x < 0 || x >= ntc) continue;
                                const int sj = S.sp[g] + j;
                                S.u.t.tri_si[x] = (unsigned short)srow;
                                S.u.t.tri_sj[x] = (unsigned short)sj;
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
                                S.u.t.cpre[x] = cnt;
                                const unsigned pos = S.pt_base + (unsigned)(tc0 + x);
                                const int dom = (int)((S.D[srow * W + (j >> 6)] >> (j & 63)) & 1ull);
                                if (pos < P.pt_cap)
                                    P.pt[pos] = make_int4(t0 + g0 + g, S.srank[srow], S.srank[sj],
                                                          (int)S.sli[srow] | (j << 16) | (dom << 31));
                            }
                        }
                    }
                    __syncthreads();
                    const int ncand = block_scan_excl(S.u.t.cpre, ntc, S.wtot);
                    // ---- D: dense over tet candidates (pipeline.py:447-479)
                    for (int c0 = 0; c0 < ncand; c0 += T2_THREADS) {
                        const int c = c0 + tid;
                        bool keep = false;
                        int4 er = make_int4(0, 0, 0, 0);
                        int el = 0;
                        if (c < ncand) {
                            const int x = owner_of(S.u.t.cpre, ntc, c);
                            const int s = S.u.t.tri_si[x], sj = S.u.t.tri_sj[x];
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
                            const int k = nth_bit_multi<W>(cm, c - S.u.t.cpre[x]);
                            const int g = S.sgen[s];
                            const int sk = S.sp[g] + k;
                            Atom au, av, aw, ax;
                            au.x = S.gx[g0 + g]; au.y = S.gy[g0 + g]; au.z = S.gz[g0 + g]; au.r2 = S.gr2[g0 + g];
                            av.x = S.sx[s]; av.y = S.sy[s]; av.z = S.sz[s]; av.r2 = S.sr2[s];
                            aw.x = S.sx[sj]; aw.y = S.sy[sj]; aw.z = S.sz[sj]; aw.r2 = S.sr2[sj];
                            ax.x = S.sx[sk]; ax.y = S.sy[sk]; ax.z = S.sz[sk]; ax.r2 = S.sr2[sk];
                            const int ou = S.gorig[g0 + g], ov = S.sorig[s], ow = S.sorig[sj], ox = S.sorig[sk];
                            const int t = t0 + g0 + g;
                            const Ortho e4 = ortho_tet(ou, au, ov, av, ow, aw, ox, ax, P.tol.eps_sing);   // pipeline.py:475-477
                            if (e4.singular) {
                                const unsigned tri_ord = (unsigned)(tc0 + x - S.rowpre[S.sp[g]]);        // ordinal among u's triangles
                                record_singular(P, make_err_key(ST_TET, t, (tri_ord << 8) | (unsigned)k), ou, ov, ow, ox, 4);
                            }
                            keep = e4.size <= P.tol.lim_a;                                               // pipeline.py:478
                            if (keep && (P.cull & 1) &&
                                dominated_by_partner(S, g, g0, s, sj, sk, e4.cx, e4.cy, e4.cz, e4.size - P.tol.eps_abs))
                                keep = false;        // AC2 would fail at this partner (it lies in the 27-cell block): never kept
                            er = make_int4(t, S.srank[s], S.srank[sj], S.srank[sk]);
                            el = (int)S.sli[s] | (j << 8) | (k << 16);
                        }
                        // block-level compaction: one global atomic per round, kept tets of a tile stay together
                        const unsigned m = __ballot_sync(FULL, keep);
                        if (lane == 0) S.qoff[tid >> 5] = __popc(m);
                        __syncthreads();
                        if (tid == 0) {
                            int tot = 0;
#pragma unroll
                            for (int w = 0; w < T2_WARPS; ++w) { const int cw = S.qoff[w]; S.qoff[w] = tot; tot += cw; }
                            S.pq_base = tot ? atomicAdd(&P.ctr->n_pq, (unsigned)tot) : 0u;
                        }
                        __syncthreads();
                        if (keep) {
                            const unsigned pos = S.pq_base + (unsigned)S.qoff[tid >> 5] + (unsigned)__popc(m & lanemask_lt());
                            if (pos < P.pq_cap) { P.pq_r[pos] = er; P.pq_l[pos] = el; }
                        }
                        __syncthreads();
                    }
                    __syncthreads();
                }
            }
            __syncthreads();
            g0 = g1;
        }
    }
}

}  // namespace axb
