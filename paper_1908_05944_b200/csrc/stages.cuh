// stages.cuh -- the standalone stage operations on caller-supplied intermediates
// (reference pipeline.py:640-731: potential_triangles(edges, ...), potential_tets(triangles, ...),
// prune(potentials, ...) consume the ROWS of the previous level) and the AC2 mask of a level
// (pipeline.py:286-313) as an operation of its own.
//
// The hot path keeps its intermediates in rank space (forward star per generator, partner slots);
// these kernels translate canonical rows of ball indices into that layout so that the same
// estimation / pruning kernels run on a level the caller handed in (possibly edited), and the one
// stage the hot path fuses differently -- the reference's standalone potential_tets, which extends
// every given triangle by a larger ball index and asks for all four faces in the given list -- as
// a kernel of its own.  None of this is on the timed path.
#pragma once

#include "common.cuh"
#include "estimate.cuh"
#include "predicates.cuh"
#include "prune.cuh"

namespace axb {

// ---- potential edges from rows (m, 2): count per generator, scatter, order every partner list by rank
__global__ void __launch_bounds__(256) k_import_edge_count(const int64_t *__restrict__ rows, unsigned m, int n,
                                                           const int *__restrict__ rank, int *__restrict__ deg,
                                                           Counters *ctr) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int64_t a = rows[2 * (size_t)e], b = rows[2 * (size_t)e + 1];
    if (a < 0 || b < 0 || a >= n || b >= n || a == b) { atomicOr(&ctr->overflow, 1u << 6); return; }
    atomicAdd(deg + min(rank[a], rank[b]), 1);
}

__global__ void __launch_bounds__(256) k_import_edge_scatter(const int64_t *__restrict__ rows, unsigned m, int n,
                                                             const int *__restrict__ rank, const uint32_t *__restrict__ adj_off,
                                                             int *__restrict__ cursor, int *__restrict__ pe_u, int *__restrict__ pe_v) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int64_t a = rows[2 * (size_t)e], b = rows[2 * (size_t)e + 1];
    if (a < 0 || b < 0 || a >= n || b >= n || a == b) return;
    const int ra = rank[a], rb = rank[b];
    const int g = min(ra, rb), p = max(ra, rb);
    const unsigned pos = adj_off[g] + (unsigned)atomicAdd(cursor + g, 1);
    pe_u[pos] = g;
    pe_v[pos] = p;
}

__global__ void __launch_bounds__(256) k_import_edge_order(int n, const uint32_t *__restrict__ adj_off, const int *__restrict__ deg,
                                                           int *__restrict__ pe_v, Counters *ctr) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned d = 0;
    if (g < n) {
        d = (unsigned)deg[g];
        int *v = pe_v + adj_off[g];
        for (unsigned a = 1; a < d; ++a) {                    // lists are short (a handful of partners)
            const int x = v[a];
            int b = (int)a - 1;
            while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; --b; }
            v[b + 1] = x;
        }
        for (unsigned a = 1; a < d; ++a)
            if (v[a] == v[a - 1]) atomicOr(&ctr->overflow, 1u << 7);     // the same edge twice
        if (d > 1) atomicAdd(&ctr->pair_bound, (unsigned long long)d * (d - 1) / 2);
    }
    unsigned md = d;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) md = max(md, __shfl_xor_sync(FULL, md, o));
    if (lane_id() == 0 && md) atomicMax(&ctr->max_deg, md);
}

// ---- potential triangles / tets from rows (m, 3) / (m, 4): ranks ascending, partner slots in the generator's list
__global__ void __launch_bounds__(256) k_import_simplices(int k, const int64_t *__restrict__ rows, unsigned m, int n,
                                                          const int *__restrict__ rank, const uint32_t *__restrict__ adj_off,
                                                          const int *__restrict__ deg, const int *__restrict__ pe_v,
                                                          int4 *__restrict__ pt, int4 *__restrict__ pq_r, int *__restrict__ pq_l,
                                                          Counters *ctr) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int r[4] = {0, 0, 0, 0};
    bool ok = true;
    for (int a = 0; a < k; ++a) {
        const int64_t v = rows[(size_t)e * k + a];
        ok = ok && v >= 0 && v < n;
        r[a] = ok ? rank[v] : 0;
    }
    sort_small(r, k);
    for (int a = 1; a < k; ++a) ok = ok && r[a] != r[a - 1];
    int s[3] = {-1, -1, -1};
    if (ok) {
        const unsigned base = adj_off[r[0]];
        const int d = deg[r[0]];
        for (int a = 1; a < k; ++a) s[a - 1] = find_partner(pe_v, base, d, r[a]);
        for (int a = 1; a < k; ++a) ok = ok && s[a - 1] >= 0;
    }
    if (!ok) {                                                // an edge of this simplex is not in the edge level
        atomicOr(&ctr->overflow, 1u << 6);
        s[0] = s[1] = s[2] = 0;
    }
    if (k == 3) {
        pt[e] = make_int4(r[0], r[1], r[2], s[0] | (s[1] << 16));
    } else {
        pq_r[e] = make_int4(r[0], r[1], r[2], r[3]);
        pq_l[e] = pack_slots(s[0], s[1], s[2]);
    }
}

// ---- the reference's standalone potential_tets (pipeline.py:670-709): every given triangle (i < j < k, ball
// indices, rows in lexicographic order) is extended by the balls x > k of the 5x5x5 cell block around ball i whose
// three new faces are all in the given list; kept if the ortho-size is at most alpha + slack.
__device__ __forceinline__ bool tri_row_less(const int64_t *__restrict__ rows, unsigned q, int64_t a, int64_t b, int64_t c) {
    const int64_t x = rows[3 * (size_t)q], y = rows[3 * (size_t)q + 1], z = rows[3 * (size_t)q + 2];
    return x < a || (x == a && (y < b || (y == b && z < c)));
}

__device__ __forceinline__ bool has_tri_row(const int64_t *__restrict__ rows, unsigned m, int64_t a, int64_t b, int64_t c) {
    unsigned lo = 0, hi = m;
    while (lo < hi) {
        const unsigned mid = (lo + hi) >> 1;
        if (tri_row_less(rows, mid, a, b, c)) lo = mid + 1; else hi = mid;
    }
    return lo < m && rows[3 * (size_t)lo] == a && rows[3 * (size_t)lo + 1] == b && rows[3 * (size_t)lo + 2] == c;
}

struct TetsFromTris {
    GridView g;
    const Atom *atoms;
    const int *orig;
    const int *rank;
    const int4 *cell_of_rank;
    const uint32_t *adj_off;
    const int *deg;
    const int *pe_v;
    const int64_t *rows;          // (m, 3)
    unsigned m;
    double lim_a, eps_sing;
    int4 *pq_r;
    int *pq_l;
    uint32_t pq_cap;
    Counters *ctr;
    ErrRecord *errs;
    unsigned long long report_key;
};

__global__ void __launch_bounds__(128) k_tets_from_triangles(TetsFromTris P) {
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.m) return;
    const int64_t bi = P.rows[3 * (size_t)t], bj = P.rows[3 * (size_t)t + 1], bk = P.rows[3 * (size_t)t + 2];
    if (bi < 0 || bk >= P.g.n || !(bi < bj && bj < bk)) { atomicOr(&P.ctr->overflow, 1u << 6); return; }
    const int ri = P.rank[bi], rj = P.rank[bj], rk = P.rank[bk];
    const Atom ai = load_atom(P.atoms, ri), aj = load_atom(P.atoms, rj), ak = load_atom(P.atoms, rk);
    const int4 cell = P.cell_of_rank[ri];
    unsigned ordinal = 0;
    for (int z = max(cell.z - 2, 0); z <= min(cell.z + 2, P.g.dz - 1); ++z)
        for (int y = max(cell.y - 2, 0); y <= min(cell.y + 2, P.g.dy - 1); ++y) {
            int s, e;
            row_range(P.g, max(cell.x - 2, 0), min(cell.x + 2, P.g.dx - 1), y, z, s, e);
            for (int rx = s; rx < e; ++rx) {
                const int64_t bx = P.orig[rx];
                if (bx <= bk) continue;
                if (!has_tri_row(P.rows, P.m, bi, bj, bx) || !has_tri_row(P.rows, P.m, bi, bk, bx) ||
                    !has_tri_row(P.rows, P.m, bj, bk, bx))
                    continue;
                const Atom p[4] = {ai, aj, ak, load_atom(P.atoms, rx)};
                const Ortho o = orthoN<4>(p, P.eps_sing);
                if (o.singular)
                    record_singular_impl(P.ctr, P.errs, P.report_key, make_err_key(ST_TET, (int)t, ordinal),
                                         (int)bi, (int)bj, (int)bk, (int)bx, 4);
                ++ordinal;
                if (!(o.size <= P.lim_a)) continue;
                int r[4] = {ri, rj, rk, rx};
                sort_small(r, 4);
                const unsigned base = P.adj_off[r[0]];
                const int d = P.deg[r[0]];
                const int s0 = find_partner(P.pe_v, base, d, r[1]), s1 = find_partner(P.pe_v, base, d, r[2]),
                          s2 = find_partner(P.pe_v, base, d, r[3]);
                if (s0 < 0 || s1 < 0 || s2 < 0) atomicOr(&P.ctr->overflow, 1u << 6);   // an edge is missing from the edge level
                const unsigned pos = atomicAdd(&P.ctr->n_pq, 1u);
                if (pos < P.pq_cap) {
                    P.pq_r[pos] = make_int4(r[0], r[1], r[2], r[3]);
                    P.pq_l[pos] = pack_slots(max(s0, 0), max(s1, 0), max(s2, 0));
                }
            }
        }
}

// ---- pipeline.py:286-313 as an operation of its own: the AC2 mask of one resident potential level
__global__ void __launch_bounds__(128) k_ac2_mask(int what, unsigned m, GridView g, Tol tol, const Atom *__restrict__ atoms,
                                                  const int *__restrict__ orig, const int *__restrict__ pe_u,
                                                  const int *__restrict__ pe_v, const int4 *__restrict__ pt,
                                                  const int4 *__restrict__ pq_r, unsigned char *__restrict__ mask) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int r[4] = {-1, -1, -1, -1};
    Ortho o;
    if (what == 0) {
        r[0] = pe_u[e]; r[1] = pe_v[e];
        o = ortho_edge(orig[r[0]], load_atom(atoms, r[0]), orig[r[1]], load_atom(atoms, r[1]), tol.eps_sing);
    } else if (what == 1) {
        const int4 q = pt[e];
        r[0] = q.x; r[1] = q.y; r[2] = q.z;
        o = ortho_tri(orig[r[0]], load_atom(atoms, r[0]), orig[r[1]], load_atom(atoms, r[1]), orig[r[2]], load_atom(atoms, r[2]),
                      tol.eps_sing);
    } else {
        const int4 q = pq_r[e];
        r[0] = q.x; r[1] = q.y; r[2] = q.z; r[3] = q.w;
        o = ortho_tet(orig[r[0]], load_atom(atoms, r[0]), orig[r[1]], load_atom(atoms, r[1]), orig[r[2]], load_atom(atoms, r[2]),
                      orig[r[3]], load_atom(atoms, r[3]), tol.eps_sing);
    }
    mask[e] = ac2_pass(g, atoms, o.cx, o.cy, o.cz, o.size - tol.eps_abs, tol.r2max, r[0], r[1], r[2], r[3]) ? 1 : 0;
}

}  // namespace axb
