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

}  // namespace axb
