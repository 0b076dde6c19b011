// heavy.cuh -- potential triangles and tets of generators with more partners than a warp tile of k_tri_tet3
// holds (more than 256: alpha of tens of A^2 at protein density).  The reference has no density limit
// (pipeline.py:373-479), so neither has this path; it is the rare, slow one: a block per generator, the two
// bit matrices ("pair is a potential edge", "pair closes a potential triangle") in global scratch, plain loops.
// Same predicates, same enumeration ordinals (error keys) and the same list entries as estimate3.cuh.
#pragma once

#include "common.cuh"
#include "estimate.cuh"
#include "predicates.cuh"

namespace axb {

constexpr int HEAVY_THREADS = 256;
constexpr int HEAVY_MIN_DEG = 257;            // k_tri_tet3<4> handles up to 64 * 4 = 256 partners per generator (its PCAP)

__global__ void __launch_bounds__(256) k_list_heavy(int lo, int hi, const int *__restrict__ deg, int *__restrict__ list,
                                                    unsigned *__restrict__ n_heavy) {
    const int t = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (t < hi && deg[t] >= HEAVY_MIN_DEG) list[atomicAdd(n_heavy, 1u)] = t;
}

// position of the nth set bit of a row of `words` 64-bit words
__device__ __forceinline__ int nth_bit_row(const unsigned long long *row, int words, int nth) {
    for (int w = 0; w < words; ++w) {
        const unsigned long long m = row[w];
        const int c = __popcll(m);
        if (nth < c) return 64 * w + nth_set_bit(m, nth);
        nth -= c;
    }
    return -1;
}

// scratch: per block 2 * (MAXP + 1) * words 64-bit words (M rows, then T rows)
__global__ void __launch_bounds__(HEAVY_THREADS) k_tri_tet_heavy(EstParams P, const int *__restrict__ heavy,
                                                                 const unsigned *__restrict__ n_heavy_dev, int words,
                                                                 unsigned long long *__restrict__ scratch) {
    __shared__ int s_rowpre[MAXP + 2];
    __shared__ unsigned s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long *M = scratch + (size_t)blockIdx.x * 2 * (MAXP + 1) * words;
    unsigned long long *T = M + (size_t)(MAXP + 1) * words;
    const unsigned n_heavy = *n_heavy_dev;
    for (unsigned h = blockIdx.x; h < n_heavy; h += gridDim.x) {
        const int t = heavy[h];
        if (t < P.own_lo && __ldg(P.pe_v + P.adj_off[t] + P.deg[t] - 1) < P.own_lo) continue;   // slab, lower halo (estimate3.cuh)
        const int d = min(P.deg[t], MAXP);
        const unsigned bu = P.adj_off[t];
        const Atom au = load_atom(P.atoms, t);
        const int ou = P.orig[t];
        for (int x = tid; x < d * words; x += HEAVY_THREADS) { M[x] = 0ull; T[x] = 0ull; }
        __syncthreads();
        // ---- partner pairs (i < j): a warp per row i, its lanes over j
        for (int i = warp; i < d; i += HEAVY_THREADS / 32) {
            const int ri = P.pe_v[bu + i];
            const Atom ai = load_atom(P.atoms, ri);
            const double rchi = P.reach[ri];
            const int oi = P.orig[ri];
            for (int j = i + 1 + lane; j < d; j += 32) {
                const int rj = P.pe_v[bu + j];
                const Atom aj = load_atom(P.atoms, rj);
                if (!reach_pair(ai, rchi, aj, P.reach[rj])) continue;                                    // pipeline.py:398-401
                const int oj = P.orig[rj];
                const unsigned q = (unsigned)(i * (2 * d - i - 1) / 2 + (j - i - 1));                    // triu ordinal
                const Ortho e2 = ortho_edge(oi, ai, oj, aj, P.tol.eps_sing);                             // pipeline.py:412-414
                if (e2.singular) record_singular(P, make_err_key(ST_VW, t, q), oi, oj, -1, -1, 2);
                if (!(e2.size <= P.tol.lim_a)) continue;                                                 // pipeline.py:415
                atomicOr(M + (size_t)i * words + (j >> 6), 1ull << (j & 63));
                atomicOr(M + (size_t)j * words + (i >> 6), 1ull << (i & 63));
                const Ortho e3 = ortho_tri(ou, au, oi, ai, oj, aj, P.tol.eps_sing);                      // pipeline.py:417-419
                if (e3.singular) record_singular(P, make_err_key(ST_TRI, t, q), ou, oi, oj, -1, 3);
                if (e3.size <= P.tol.lim_a) atomicOr(T + (size_t)i * words + (j >> 6), 1ull << (j & 63));   // pipeline.py:420
            }
        }
        __threadfence();
        __syncthreads();
        // ---- triangle numbering: row counts, prefix, one reservation in the global list
        for (int i = tid; i < d; i += HEAVY_THREADS) {
            int c = 0;
            for (int w = 0; w < words; ++w) c += __popcll(T[(size_t)i * words + w]);
            s_rowpre[i] = c;
        }
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int i = 0; i < d; ++i) { const int c = s_rowpre[i]; s_rowpre[i] = run; run += c; }
            s_rowpre[d] = run;
            s_base = run ? atomicAdd(&P.ctr->n_pt, (unsigned)run) : 0u;
        }
        __syncthreads();
        const int ntri = s_rowpre[d];
        // ---- a thread per triangle: list entry, then its tet candidates (pipeline.py:447-479)
        for (int x = tid; x < ntri; x += HEAVY_THREADS) {
            int lo = 0, hi = d;                            // last row whose prefix does not exceed x
            while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (s_rowpre[mid] <= x) lo = mid; else hi = mid; }
            const int i = lo;
            const int j = nth_bit_row(T + (size_t)i * words, words, x - s_rowpre[i]);
            const int ri = P.pe_v[bu + i], rj = P.pe_v[bu + j];
            const unsigned pos = s_base + (unsigned)x;
            if (pos < P.pt_cap) P.pt[pos] = make_int4(t, ri, rj, i | (j << 16));
            const Atom ai = load_atom(P.atoms, ri), aj = load_atom(P.atoms, rj);
            const int oi = P.orig[ri], oj = P.orig[rj];
            for (int w = j >> 6; w < words; ++w) {
                unsigned long long m = M[(size_t)i * words + w] & M[(size_t)j * words + w];
                if (w == (j >> 6)) m &= (j & 63) == 63 ? 0ull : (~0ull << ((j & 63) + 1));              // partners above j only
                while (m) {
                    const int k = 64 * w + __ffsll((long long)m) - 1;
                    m &= m - 1;
                    const int rk = P.pe_v[bu + k];
                    const int ok = P.orig[rk];
                    const Ortho e4 = ortho_tet(ou, au, oi, ai, oj, aj, ok, load_atom(P.atoms, rk), P.tol.eps_sing);   // pipeline.py:475-477
                    if (e4.singular) record_singular(P, make_err_key(ST_TET, t, tet_ordinal((unsigned)x, k)), ou, oi, oj, ok, 4);
                    if (!(e4.size <= P.tol.lim_a)) continue;                                             // pipeline.py:478
                    const unsigned at = atomicAdd(&P.ctr->n_pq, 1u);
                    if (at < P.pq_cap) { P.pq_r[at] = make_int4(t, ri, rj, rk); P.pq_l[at] = pack_slots(i, j, k); }
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace axb
