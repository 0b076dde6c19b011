// sweep.cuh -- alpha sweep with re-use (the paper's stated future work, PAPER.md:469:
// "utilize a previously computed alpha complex to efficiently compute the alpha complex for higher values of alpha").
//
// What depends on alpha in the reference pipeline is only WHICH simplices are looked at:
//   * the reach pre-filter of a pair (pipeline.py:322-324, 341-344, 398-401) and the tests `size <= alpha + eps`
//     (pipeline.py:358, 415, 420, 478) -- both monotone in alpha, so every potential simplex at alpha is in the
//     lists built at a larger alpha;
//   * ortho-centres, ortho-sizes and the domination check AC2 (pipeline.py:286-313) are functions of the simplex
//     and the ball set alone.
// So the grid, the potential lists, the ortho solves and ALL AC2 walks are done once at the largest alpha of the
// sweep (k_sweep_prepare_*); per alpha there remain a flag per listed edge (k_sweep_edge_flags: the very same
// pre-filter and size comparison, re-evaluated with that alpha's reach and limit), the inheritance marks of the
// pruning kernels (prune.cuh, sweep mode: array look-ups instead of solves and walks) and the canonical lists.
// Bit-exact with an independent run at each alpha: every comparison is the reference's, on the same fp64 values.
#pragma once

#include "common.cuh"
#include "predicates.cuh"
#include "estimate.cuh"
#include "prune.cuh"

namespace axb {

struct SweepArrays {
    double *esize;                 // (n_pe) ortho-size per listed edge
    unsigned char *pf;             // (n_pe) potential at the current alpha
    double *tsize;                 // (n_pt)
    int *tvw;                      // (n_pt)
    double *qsize, *qtsize;        // (n_pq)
    int4 *qe;                      // (n_pq)
    unsigned char *ac2e, *ac2t, *ac2q;
    // ranked sweep (below): per listed simplex the index of the first alpha of the sweep at which it is kept
    unsigned char *ke;             // (n_pe) first alpha index at which the edge is potential (K = never)
    unsigned *ae, *at, *aq, *av;   // (n_pe) (n_pt) (n_pq) (n) first alpha index at which the simplex is KEPT
    unsigned long long *ptmask;    // (n_pe, W) listed triangles by (row, partner bit)
    unsigned *row_first;           // (n_pe) list position of the row's first triangle
    const double *alphas;          // (K) ascending, on the device
    int K;
};

constexpr int SWEEP_THREADS = 128;

__global__ void __launch_bounds__(SWEEP_THREADS) k_sweep_prepare_edges(PruneParams P, unsigned m, SweepArrays S) {
    __shared__ int2 s_rows[9][SWEEP_THREADS];
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int u = P.pe_u[e], v = P.pe_v[e];
    const Ortho o = ortho_edge(P.orig[u], load_atom(P.atoms, u), P.orig[v], load_atom(P.atoms, v), P.tol.eps_sing);
    S.esize[e] = o.size;
    S.ac2e[e] = ac2_check(P, o.cx, o.cy, o.cz, o.size - P.tol.eps_abs, u, v, -1, -1, &s_rows[0][threadIdx.x], SWEEP_THREADS) ? 1 : 0;
}

__global__ void __launch_bounds__(SWEEP_THREADS) k_sweep_prepare_tris(PruneParams P, unsigned m, SweepArrays S) {
    __shared__ int2 s_rows[9][SWEEP_THREADS];
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int4 r = P.pt[e];
    const Ortho o = ortho_tri(P.orig[r.x], load_atom(P.atoms, r.x), P.orig[r.y], load_atom(P.atoms, r.y), P.orig[r.z],
                              load_atom(P.atoms, r.z), P.tol.eps_sing);
    S.tsize[e] = o.size;
    const unsigned bv = P.adj_off[r.y];
    const int iw = find_partner(P.pe_v, bv, P.deg[r.y], r.z);
    if (iw < 0) note_miss(P);
    S.tvw[e] = (int)bv + max(iw, 0);
    S.ac2t[e] = ac2_check(P, o.cx, o.cy, o.cz, o.size - P.tol.eps_abs, r.x, r.y, r.z, -1, &s_rows[0][threadIdx.x], SWEEP_THREADS) ? 1 : 0;
}

__global__ void __launch_bounds__(SWEEP_THREADS) k_sweep_prepare_tets(PruneParams P, unsigned m, SweepArrays S) {
    __shared__ int2 s_rows[9][SWEEP_THREADS];
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int4 r = P.pq_r[e];
    const Atom au = load_atom(P.atoms, r.x), av = load_atom(P.atoms, r.y), aw = load_atom(P.atoms, r.z), ax = load_atom(P.atoms, r.w);
    const int ou = P.orig[r.x], ov = P.orig[r.y], ow = P.orig[r.z], ox = P.orig[r.w];
    const Ortho o = ortho_tet(ou, au, ov, av, ow, aw, ox, ax, P.tol.eps_sing);
    S.qsize[e] = o.size;
    S.qtsize[e] = ortho_tri(ou, au, ov, av, ow, aw, P.tol.eps_sing).size;       // the triangle the tet was grown from
    const unsigned bv = P.adj_off[r.y], bw = P.adj_off[r.z];
    const int dv = P.deg[r.y];
    const int iw = find_partner(P.pe_v, bv, dv, r.z), ix = find_partner(P.pe_v, bv, dv, r.w);
    const int jx = find_partner(P.pe_v, bw, P.deg[r.z], r.w);
    if (iw < 0 || ix < 0 || jx < 0) note_miss(P);
    S.qe[e] = make_int4((int)bv + max(iw, 0), (int)bv + max(ix, 0), (int)bw + max(jx, 0), 0);
    S.ac2q[e] = ac2_check(P, o.cx, o.cy, o.cz, o.size - P.tol.eps_abs, r.x, r.y, r.z, r.w, &s_rows[0][threadIdx.x], SWEEP_THREADS) ? 1 : 0;
}

// pipeline.py:322-324 (reach, viability), 341-344 (pre-filter), 358 (size test) of one listed edge at `alpha`
__global__ void __launch_bounds__(256) k_sweep_edge_flags(unsigned m, const Atom *__restrict__ atoms, const int *__restrict__ pe_u,
                                                          const int *__restrict__ pe_v, const double *__restrict__ esize,
                                                          double alpha, double eps_abs, unsigned char *__restrict__ pf) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const Atom a = load_atom(atoms, pe_u[e]), b = load_atom(atoms, pe_v[e]);
    const double la = a.r2 + alpha + eps_abs, lb = b.r2 + alpha + eps_abs;
    bool ok = la >= 0.0 && lb >= 0.0;
    if (ok) {
        const double ra = sqrt(fmax(la, 0.0)), rb = sqrt(fmax(lb, 0.0));
        const double dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
        const double lims = rb + ra;
        ok = (dx * dx + dy * dy) + dz * dz <= lims * lims && esize[e] <= alpha + eps_abs;
    }
    pf[e] = ok ? 1 : 0;
}

// ---------------------------------------------------------------------------------------------------------------
// Ranked sweep.  With the alphas of the sweep known up front (ascending, K of them) every listed simplex gets the index
// of the first alpha at which the reference keeps it:
//     own(s)  = first k with "s is potential at alpha_k" (the flags above, each evaluated with alpha_k's reach and limit;
//               they are monotone in alpha), if AC2(s) holds, else K (never);
//     a(s)    = min(own(s), min over the listed cofaces t of s of a(t))          (inheritance, pipeline.py:501-513)
// computed once, top-down (tets -> triangles -> edges -> vertices, atomicMin).  The complex at alpha_k is then
// { s : a(s) <= k }: a threshold pass per alpha instead of the pruning kernels' scans.  Needs every face of a listed
// tet to be a listed triangle (true unless rounding puts a face's size above its tet's; checked, else the caller uses
// axb_sweep_prune).

__device__ __forceinline__ int first_alpha_with_size(const SweepArrays &S, double size, double eps_abs) {
    int k = 0;
    while (k < S.K && !(size <= S.alphas[k] + eps_abs)) ++k;
    return k;
}

// list position of the triangle (row e, partner bit j); -1 if it is not listed
__device__ __forceinline__ int listed_triangle(const SweepArrays &S, int W, unsigned e, int j) {
    const unsigned long long *row = S.ptmask + (size_t)e * W;
    if (!((row[j >> 6] >> (j & 63)) & 1ull)) return -1;
    int below = 0;
    for (int w = 0; w < (j >> 6); ++w) below += __popcll(row[w]);
    below += __popcll(row[j >> 6] & ((1ull << (j & 63)) - 1ull));
    return (int)S.row_first[e] + below;                          // a row's triangles are contiguous, ascending in j
}

__global__ void __launch_bounds__(256) k_sweep_tri_index(PruneParams P, unsigned m, SweepArrays S) {
    const unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m) return;
    const int4 r = P.pt[x];
    const int i = r.w & 0xffff, j = (r.w >> 16) & 0x7fff;
    const unsigned e = P.adj_off[r.x] + (unsigned)i;
    atomicOr(S.ptmask + (size_t)e * P.W + (j >> 6), 1ull << (j & 63));
    atomicMin(S.row_first + e, x);
}

__global__ void __launch_bounds__(256) k_sweep_rank_edges(PruneParams P, unsigned m, SweepArrays S) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const Atom a = load_atom(P.atoms, P.pe_u[e]), b = load_atom(P.atoms, P.pe_v[e]);
    const double dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    const double d2 = (dx * dx + dy * dy) + dz * dz;
    const double size = S.esize[e];
    int k = 0;
    for (; k < S.K; ++k) {                                        // pipeline.py:322-324, 341-344, 358 at alpha_k
        const double alpha = S.alphas[k];
        const double la = a.r2 + alpha + P.tol.eps_abs, lb = b.r2 + alpha + P.tol.eps_abs;
        if (!(la >= 0.0 && lb >= 0.0)) continue;
        const double lims = sqrt(fmax(lb, 0.0)) + sqrt(fmax(la, 0.0));
        if (d2 <= lims * lims && size <= alpha + P.tol.eps_abs) break;
    }
    S.ke[e] = (unsigned char)k;
    S.ae[e] = S.ac2e[e] ? (unsigned)k : (unsigned)S.K;
}

__global__ void __launch_bounds__(256) k_sweep_rank_tris(PruneParams P, unsigned m, SweepArrays S) {
    const unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m) return;
    const int4 r = P.pt[x];
    const int i = r.w & 0xffff, j = (r.w >> 16) & 0x7fff;
    const unsigned bu = P.adj_off[r.x];
    int k = max(max((int)S.ke[bu + i], (int)S.ke[bu + j]), (int)S.ke[S.tvw[x]]);              // pipeline.py:398-415
    k = max(k, first_alpha_with_size(S, S.tsize[x], P.tol.eps_abs));                          // pipeline.py:420
    S.at[x] = S.ac2t[x] ? (unsigned)k : (unsigned)S.K;
}

__global__ void __launch_bounds__(256) k_sweep_rank_tets(PruneParams P, unsigned m, SweepArrays S) {
    const unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m) return;
    const int4 r = P.pq_r[x];
    const int l = P.pq_l[x];
    const int i = l & SLOT_MASK, j = (l >> SLOT_BITS) & SLOT_MASK, kk = (l >> (2 * SLOT_BITS)) & SLOT_MASK;
    const unsigned bu = P.adj_off[r.x];
    const int4 qe = S.qe[x];
    int k = max(max((int)S.ke[bu + i], (int)S.ke[bu + j]), (int)S.ke[bu + kk]);
    k = max(k, max(max((int)S.ke[qe.x], (int)S.ke[qe.y]), (int)S.ke[qe.z]));                  // pipeline.py:447-466
    k = max(k, first_alpha_with_size(S, S.qtsize[x], P.tol.eps_abs));
    k = max(k, first_alpha_with_size(S, S.qsize[x], P.tol.eps_abs));                          // pipeline.py:478
    const unsigned a = S.ac2q[x] ? (unsigned)min(k, S.K) : (unsigned)S.K;
    S.aq[x] = a;
    if (a >= (unsigned)S.K) return;
    // its four faces inherit it: (u; i, j), (u; i, k), (u; j, k) in u's rows, (v; w, x) in v's
    const unsigned bv = P.adj_off[r.y];
    const int iw = qe.x - (int)bv, ix = qe.y - (int)bv;
    const int f0 = listed_triangle(S, P.W, bu + i, j), f1 = listed_triangle(S, P.W, bu + i, kk);
    const int f2 = listed_triangle(S, P.W, bu + j, kk), f3 = listed_triangle(S, P.W, bv + iw, ix);
    if (f0 < 0 || f1 < 0 || f2 < 0 || f3 < 0) { atomicOr(&P.ctr->overflow, 1u << 8); return; }
    atomicMin(S.at + f0, a); atomicMin(S.at + f1, a); atomicMin(S.at + f2, a); atomicMin(S.at + f3, a);
}

__global__ void __launch_bounds__(256) k_sweep_inherit_tris(PruneParams P, unsigned m, SweepArrays S) {
    const unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m) return;
    const unsigned a = S.at[x];
    if (a >= (unsigned)S.K) return;
    const int4 r = P.pt[x];
    const int i = r.w & 0xffff, j = (r.w >> 16) & 0x7fff;
    const unsigned bu = P.adj_off[r.x];
    atomicMin(S.ae + bu + i, a); atomicMin(S.ae + bu + j, a); atomicMin(S.ae + S.tvw[x], a);
}

__global__ void __launch_bounds__(256) k_sweep_inherit_edges(PruneParams P, unsigned m, SweepArrays S) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const unsigned a = S.ae[e];
    if (a >= (unsigned)S.K) return;
    atomicMin(S.av + P.pe_u[e], a); atomicMin(S.av + P.pe_v[e], a);
}

// pipeline.py:517-525: a vertex is kept with an incident kept edge, or on its own (biomolecule mode, or a non-dominated
// ball whose size -r^2 is within the limit)
__global__ void __launch_bounds__(256) k_sweep_rank_vertices(PruneParams P, SweepArrays S) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.g.n) return;
    unsigned own = (unsigned)S.K;
    if (P.biomolecule) {
        own = 0u;
    } else {
        const Atom a = load_atom(P.atoms, t);
        const int k = first_alpha_with_size(S, -a.r2, P.tol.eps_abs);
        if (k < S.K && ac2_pass(P.g, P.atoms, a.x, a.y, a.z, -a.r2 - P.tol.eps_abs, P.tol.r2max, t, -1, -1, -1)) own = (unsigned)k;
    }
    atomicMin(S.av + t, own);
}

// ---- the complex at alpha_k: everything with a first-kept index <= k, into the pruning stage's kept-state layout
__global__ void __launch_bounds__(256) k_sweep_select(PruneParams P, SweepArrays S, unsigned k, unsigned E, unsigned T, unsigned Q) {
    const unsigned stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (unsigned x = t0; x < Q; x += stride) {
        if (S.aq[x] > k) continue;
        const int4 r = P.pq_r[x];
        int row[4] = {__ldg(P.orig + r.x), __ldg(P.orig + r.y), __ldg(P.orig + r.z), __ldg(P.orig + r.w)};
        sort_small(row, 4);
        const unsigned slot = atomicAdd(&P.ctr->n_k3, 1u);
        if (slot < P.k3_cap) P.k3[slot] = make_int4(row[0], row[1], row[2], row[3]);
        atomicAdd(P.cnt3 + row[0], 1u);
    }
    for (unsigned x = t0; x < T; x += stride) {
        if (S.at[x] > k) continue;
        const int4 r = P.pt[x];
        const int i = r.w & 0xffff, j = (r.w >> 16) & 0x7fff;
        atomicOr(P.trimask + (size_t)(P.adj_off[r.x] + i) * P.W + (j >> 6), 1ull << (j & 63));
        atomicAdd(P.cnt2 + min3(__ldg(P.orig + r.x), __ldg(P.orig + r.y), __ldg(P.orig + r.z)), 1u);
    }
    for (unsigned e = t0; e < E; e += stride) {
        if (S.ae[e] > k) continue;
        P.eflag[e] = 1u;
        atomicAdd(P.cnt1 + min(__ldg(P.orig + P.pe_u[e]), __ldg(P.orig + P.pe_v[e])), 1u);
    }
    for (unsigned t = t0; t < (unsigned)P.g.n; t += stride) P.vkeep[__ldg(P.orig + t)] = S.av[t] <= k ? 1u : 0u;
}

}  // namespace axb
