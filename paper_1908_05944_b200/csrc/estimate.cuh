// estimate.cuh -- stage one: potential edges, triangles and tetrahedra
// (reference pipeline.py:316-479), one warp per generator ball.
//
// A generator is the minimum-RANK vertex of a simplex (pipeline.py:10-15).
//   k_edges    : scans the upper half of the generator's 5x5x5 cell block --
//                13 rows of cells, each a contiguous rank range -- lanes over
//                candidates, reach pre-filter + ortho-size test, warp-ballot
//                compaction into the generator's partner list (ascending rank).
//   k_tri_tet  : stages the partner atoms in shared memory, tests all partner
//                pairs (bit matrix M of "is a potential edge"), derives the
//                potential triangles (bit matrix T) and extends each triangle
//                by the higher partners that are M-adjacent to both its
//                vertices (potential tets).
// Variable-length outputs go through warp-private shared-memory staging
// buffers that are flushed with ONE global atomicAdd per flush.
#pragma once

#include "common.cuh"
#include "predicates.cuh"

namespace axb {

constexpr int EST_WARPS = 8;
constexpr int EBUF = 512;      // partner ranks staged per warp
constexpr int EGEN = 32;       // generators staged per warp
constexpr int MAXP = 256;      // AXB_MAX_PARTNERS
constexpr int EST_TILE = 64;   // consecutive ranks handled by one block at a time
constexpr int ROWOF_CAP = 128; // candidates per generator covered by the stamped row table

struct EstParams {
    GridView g;
    Tol tol;
    const Atom *atoms;
    const double *reach;
    const int *orig;            // ball index per rank
    const int4 *cell_of_rank;   // (cx, cy, cz, key) per rank
    uint32_t *adj_off;          // per rank: start of the partner list in pe_v
    int *deg;                   // per rank: number of partners (pre-zeroed)
    int *pe_v;                  // partner rank per potential edge
    int *pe_u;                  // generator rank per potential edge
    uint32_t pe_cap;
    int4 *pt;                   // potential triangles {u, v, w, i | j << 16}
    uint32_t pt_cap;
    int4 *pq_r;                 // potential tets, ranks {u, v, w, x}
    int *pq_l;                  // potential tets, partner slots i | j << 8 | k << 16
    uint32_t pq_cap;
    Counters *ctr;
    ErrRecord *errs;
    unsigned long long report_key;   // != 0: only the solve with this key writes errs[0]
};

__device__ __forceinline__ void sort_small(int *v, int k) {
    for (int a = 1; a < k; ++a) {
        int x = v[a], b = a - 1;
        while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; --b; }
        v[b + 1] = x;
    }
}

__device__ __noinline__ void record_singular(const EstParams &P, unsigned long long key, int v0, int v1, int v2, int v3,
                                             int nv) {
    atomicMin(&P.ctr->err_key, key);
    ErrRecord r;
    r.key = key;
    r.verts[0] = v0; r.verts[1] = v1; r.verts[2] = v2; r.verts[3] = v3;
    sort_small(r.verts, nv);
    r.nverts = nv;
    r.pad = 0;
    if (P.report_key) {
        if (key == P.report_key) P.errs[0] = r;
    } else {
        unsigned slot = atomicAdd(&P.ctr->err_count, 1u);
        if (slot < ERR_CAP) P.errs[slot] = r;
    }
}

// ---------------------------------------------------------------- k_edges
__global__ void __launch_bounds__(EST_WARPS * 32, 4) k_edges(EstParams P, int rank_lo, int rank_hi) {
    __shared__ int s_buf[EST_WARPS][EBUF];
    __shared__ int s_gen[EST_WARPS][EGEN];
    __shared__ int s_goff[EST_WARPS][EGEN + 1];
    __shared__ int s_rs[EST_WARPS][16];
    __shared__ int s_rp[EST_WARPS][16];
    __shared__ unsigned char s_rowof[EST_WARPS][ROWOF_CAP];   // candidate number -> row (stamped by the row lanes)
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const GridView &g = P.g;
    int nbuf = 0, ngen = 0;                 // warp-uniform staging state
    unsigned max_deg = 0;
    unsigned long long pairs = 0;

    auto flush = [&]() {
        if (ngen == 0) return;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&P.ctr->n_pe, (unsigned)nbuf);
        base = __shfl_sync(FULL, base, 0);
        if ((unsigned long long)base + (unsigned)nbuf <= P.pe_cap) {
            if (lane == 0) s_goff[warp][ngen] = nbuf;
            __syncwarp();
            if (lane < ngen) {
                int t = s_gen[warp][lane];
                P.adj_off[t] = base + (unsigned)s_goff[warp][lane];
                P.deg[t] = s_goff[warp][lane + 1] - s_goff[warp][lane];
            }
            for (int idx = lane; idx < nbuf; idx += 32) {
                int gi = 0;                                 // last staged generator with goff <= idx
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (gi + step < ngen && s_goff[warp][gi + step] <= idx) gi += step;
                P.pe_v[base + idx] = s_buf[warp][idx];
                P.pe_u[base + idx] = s_gen[warp][gi];
            }
        } else if (lane == 0) {
            atomicOr(&P.ctr->overflow, 1u << 4);           // potential-edge buffer too small: caller re-runs
        }
        __syncwarp();
        nbuf = 0;
        ngen = 0;
    };

    const int ntiles = (rank_hi - rank_lo + EST_TILE - 1) / EST_TILE;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int t_end = min(rank_lo + (tile + 1) * EST_TILE, rank_hi);
        for (int t = rank_lo + tile * EST_TILE + warp; t < t_end; t += EST_WARPS) {
            const double ru = __ldg(P.reach + t);
            if (!(ru >= 0.0)) continue;                     // not viable (pipeline.py:336-337)
            const Atom au = load_atom(P.atoms, t);
            const int ou = __ldg(P.orig + t);
            const int4 cell = __ldg(P.cell_of_rank + t);
            const int cx = cell.x, cy = cell.y, cz = cell.z;
            // the 13 rows of the 5x5x5 block whose balls can out-rank t (pipeline.py:332-338)
            int rs = 0, rc = 0;
            if (lane < 13) {
                int oy, oz;
                if (lane < 3) { oy = lane; oz = 0; }
                else { int q = lane - 3; oz = 1 + q / 5; oy = q % 5 - 2; }
                int y = cy + oy, z = cz + oz;
                if (y >= 0 && y < g.dy && z < g.dz) {
                    int row = g.dx * (y + g.dy * z);
                    int x0 = max(cx - 2, 0), x1 = min(cx + 2, g.dx - 1);
                    int s = (int)__ldg(g.cell_start + row + x0);
                    int e = (int)__ldg(g.cell_start + row + x1 + 1);
                    if (lane == 0) s = t + 1;               // own row: only ranks above t
                    rs = s;
                    rc = max(e - s, 0);
                }
            }
            const int incl = warp_incl_scan(rc);
            const int total = __shfl_sync(FULL, incl, 31);
            if (total == 0) continue;
            if (nbuf + min(total, MAXP) > EBUF || ngen == EGEN) flush();
            __syncwarp();
            if (lane < 16) { s_rs[warp][lane] = rs; s_rp[warp][lane] = incl - rc; }
            if (lane < 13) {                                // stamp: candidate number -> row
                const int pe = min(incl, ROWOF_CAP);
                for (int p = incl - rc; p < pe; ++p) s_rowof[warp][p] = (unsigned char)lane;
            }
            __syncwarp();
            int deg = 0;
            for (int p0 = 0; p0 < total; p0 += 32) {
                const int p = p0 + lane;
                bool keep = false;
                int cand = -1;
                if (p < total) {
                    int r;
                    if (p < ROWOF_CAP) {
                        r = s_rowof[warp][p];
                    } else {
                        r = 0;
#pragma unroll
                        for (int k = 1; k < 13; ++k) r += (s_rp[warp][k] <= p) ? 1 : 0;
                    }
                    cand = s_rs[warp][r] + (p - s_rp[warp][r]);
                    const double rv = __ldg(P.reach + cand);
                    const Atom av = load_atom(P.atoms, cand);
                    if (rv >= 0.0 && reach_pair(av, rv, au, ru)) {            // pipeline.py:341-344
                        const int ov = __ldg(P.orig + cand);
                        const Ortho o = ortho_edge(ou, au, ov, av, P.tol.eps_sing);   // pipeline.py:355-356
                        if (o.singular) record_singular(P, make_err_key(ST_EDGE, t, (unsigned)p), ou, ov, -1, -1, 2);
                        keep = o.size <= P.tol.lim_a;                          // pipeline.py:358
                    }
                }
                const unsigned m = __ballot_sync(FULL, keep);
                if (keep) {
                    int slot = deg + __popc(m & lanemask_lt());
                    if (slot < MAXP) s_buf[warp][nbuf + slot] = cand;
                }
                deg += __popc(m);
            }
            if (deg > MAXP) {
                if (lane == 0) atomicOr(&P.ctr->overflow, 1u);                 // AXB_ERR_DENSITY
                deg = MAXP;
            }
            if (deg > 0) {
                if (lane == 0) { s_gen[warp][ngen] = t; s_goff[warp][ngen] = nbuf; }
                nbuf += deg;
                ngen += 1;
                max_deg = max(max_deg, (unsigned)deg);
                pairs += (unsigned long long)deg * (unsigned)(deg - 1) / 2;
            }
            __syncwarp();
        }
    }
    flush();
    if (lane == 0) {
        atomicMax(&P.ctr->max_deg, max_deg);
        atomicAdd(&P.ctr->pair_bound, pairs);
    }
}

// -------------------------------------------------------------- k_tri_tet
constexpr int TBUF = 128;   // staged potential triangles per warp
constexpr int QBUF = 128;   // staged potential tets per warp

template <int W>
struct TriWarpSmem {
    static constexpr int PCAP = 64 * W;
    double x[PCAP], y[PCAP], z[PCAP], r2[PCAP], reach[PCAP];
    unsigned long long M[PCAP * W];      // M[i] bit j: (P_i, P_j) passes reach filter and ortho-size test
    unsigned long long T[PCAP * W];      // T[i] bit j (j > i): (u, P_i, P_j) is a potential triangle
    int orig[PCAP];
    int rank[PCAP];
    int rowpre[PCAP + 1];
    int4 tbuf[TBUF];
    int4 qbuf_r[QBUF];
    int qbuf_l[QBUF];
};

__device__ __forceinline__ int nth_set_bit(unsigned long long m, int n) {
    for (int q = 0; q < n; ++q) m &= m - 1;
    return __ffsll((long long)m) - 1;
}

template <int W>
__global__ void __launch_bounds__(W == 1 ? 256 : 128) k_tri_tet(EstParams P, int rank_lo, int rank_hi) {
    constexpr int WARPS = (W == 1) ? 8 : 4;
    constexpr int PCAP = 64 * W;
    extern __shared__ __align__(16) unsigned char s_raw[];
    TriWarpSmem<W> &S = reinterpret_cast<TriWarpSmem<W> *>(s_raw)[threadIdx.x >> 5];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    int ntb = 0, nqb = 0;                   // warp-uniform staging fill

    auto flush_t = [&]() {
        if (ntb == 0) return;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&P.ctr->n_pt, (unsigned)ntb);
        base = __shfl_sync(FULL, base, 0);
        __syncwarp();
        if ((unsigned long long)base + (unsigned)ntb <= P.pt_cap) {
            for (int idx = lane; idx < ntb; idx += 32) P.pt[base + idx] = S.tbuf[idx];
        } else if (lane == 0) {
            atomicOr(&P.ctr->overflow, 1u << 1);
        }
        __syncwarp();
        ntb = 0;
    };
    auto flush_q = [&]() {
        if (nqb == 0) return;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&P.ctr->n_pq, (unsigned)nqb);
        base = __shfl_sync(FULL, base, 0);
        __syncwarp();
        if ((unsigned long long)base + (unsigned)nqb <= P.pq_cap) {
            for (int idx = lane; idx < nqb; idx += 32) {
                P.pq_r[base + idx] = S.qbuf_r[idx];
                P.pq_l[base + idx] = S.qbuf_l[idx];
            }
        } else if (lane == 0) {
            atomicOr(&P.ctr->overflow, 1u << 2);
        }
        __syncwarp();
        nqb = 0;
    };

    const int ntiles = (rank_hi - rank_lo + EST_TILE - 1) / EST_TILE;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int t_end = min(rank_lo + (tile + 1) * EST_TILE, rank_hi);
        for (int t = rank_lo + tile * EST_TILE + warp; t < t_end; t += WARPS) {
            const int d = min(__ldg(P.deg + t), PCAP);
            if (d < 2) continue;
            const unsigned abase = __ldg(P.adj_off + t);
            const Atom au = load_atom(P.atoms, t);
            const int ou = __ldg(P.orig + t);
            // ---- stage the partner atoms (ascending rank = pipeline.py:362-370 order)
            for (int i = lane; i < d; i += 32) {
                int rk = __ldg(P.pe_v + abase + i);
                Atom a = load_atom(P.atoms, rk);
                S.x[i] = a.x; S.y[i] = a.y; S.z[i] = a.z; S.r2[i] = a.r2;
                S.reach[i] = __ldg(P.reach + rk);
                S.orig[i] = __ldg(P.orig + rk);
                S.rank[i] = rk;
#pragma unroll
                for (int w = 0; w < W; ++w) { S.M[i * W + w] = 0ull; S.T[i * W + w] = 0ull; }
            }
            __syncwarp();
            // ---- all partner pairs in np.triu_indices order (pipeline.py:393-401)
            const int npairs = d * (d - 1) / 2;
            for (int p0 = 0; p0 < npairs; p0 += 32) {
                const int p = p0 + lane;
                if (p < npairs) {
                    const float b2 = (float)(2 * d - 1);
                    int i = (int)((b2 - sqrtf(b2 * b2 - 8.0f * (float)p)) * 0.5f);
                    i = max(0, min(i, d - 2));
                    while (i > 0 && i * (2 * d - i - 1) / 2 > p) --i;
                    while ((i + 1) * (2 * d - i - 2) / 2 <= p) ++i;
                    const int j = p - i * (2 * d - i - 1) / 2 + i + 1;
                    Atom av, aw;
                    av.x = S.x[i]; av.y = S.y[i]; av.z = S.z[i]; av.r2 = S.r2[i];
                    aw.x = S.x[j]; aw.y = S.y[j]; aw.z = S.z[j]; aw.r2 = S.r2[j];
                    if (reach_pair(av, S.reach[i], aw, S.reach[j])) {                    // pipeline.py:398-401
                        const int ov = S.orig[i], ow = S.orig[j];
                        const Ortho e2 = ortho_edge(ov, av, ow, aw, P.tol.eps_sing);     // pipeline.py:412-414
                        if (e2.singular) record_singular(P, make_err_key(ST_VW, t, (unsigned)p), ov, ow, -1, -1, 2);
                        if (e2.size <= P.tol.lim_a) {                                    // pipeline.py:415
                            atomicOr(&S.M[i * W + (j >> 6)], 1ull << (j & 63));
                            atomicOr(&S.M[j * W + (i >> 6)], 1ull << (i & 63));
                            const Ortho e3 = ortho_tri(ou, au, ov, av, ow, aw, P.tol.eps_sing);   // pipeline.py:417-419
                            if (e3.singular) record_singular(P, make_err_key(ST_TRI, t, (unsigned)p), ou, ov, ow, -1, 3);
                            if (e3.size <= P.tol.lim_a)                                  // pipeline.py:420
                                atomicOr(&S.T[i * W + (j >> 6)], 1ull << (j & 63));
                        }
                    }
                }
            }
            __syncwarp();
            // ---- prefix of triangles per row
            int carry = 0;
            for (int i0 = 0; i0 < d; i0 += 32) {
                const int i = i0 + lane;
                int c = 0;
                if (i < d) {
#pragma unroll
                    for (int w = 0; w < W; ++w) c += __popcll(S.T[i * W + w]);
                }
                const int incl = warp_incl_scan(c);
                if (i < d) S.rowpre[i] = carry + incl - c;
                carry += __shfl_sync(FULL, incl, 31);
            }
            const int ntri = carry;
            if (lane == 0) S.rowpre[d] = ntri;
            __syncwarp();
            if (ntri == 0) continue;
            // ---- lanes over triangles: emit the triangle, then extend it (pipeline.py:447-479)
            for (int tt0 = 0; tt0 < ntri; tt0 += 32) {
                const int tt = tt0 + lane;
                const bool valid = tt < ntri;
                int i = 0, j = 0;
                unsigned long long cand[W];
#pragma unroll
                for (int w = 0; w < W; ++w) cand[w] = 0ull;
                if (valid) {
                    int lo = 0, hi = d;                     // last row with rowpre <= tt
                    while (hi - lo > 1) {
                        int mid = (lo + hi) >> 1;
                        if (S.rowpre[mid] <= tt) lo = mid; else hi = mid;
                    }
                    i = lo;
                    int nth = tt - S.rowpre[i];
                    j = -1;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        unsigned long long m = S.T[i * W + w];
                        int c = __popcll(m);
                        if (j < 0) {
                            if (nth < c) j = 64 * w + nth_set_bit(m, nth);
                            else nth -= c;
                        }
                    }
                    // partners above j adjacent (in M) to both P_i and P_j: rank[x] > rank_hi (pipeline.py:447)
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        unsigned long long m = S.M[i * W + w] & S.M[j * W + w];
                        int lowbit = j + 1 - 64 * w;        // keep bits >= lowbit
                        if (lowbit >= 64) m = 0ull;
                        else if (lowbit > 0) m &= ~0ull << lowbit;
                        cand[w] = m;
                    }
                }
                // stage the triangles of this round
                {
                    const int cnt = min(32, ntri - tt0);
                    if (ntb + cnt > TBUF) flush_t();
                    if (valid) S.tbuf[ntb + lane] = make_int4(t, S.rank[i], S.rank[j], i | (j << 16));
                    ntb += cnt;
                    __syncwarp();
                }
                // extend: every lane walks its own candidate bits; rounds are warp-synchronous
                for (;;) {
                    int k = -1;
#pragma unroll
                    for (int w = 0; w < W; ++w)
                        if (k < 0 && cand[w]) { k = 64 * w + __ffsll((long long)cand[w]) - 1; cand[w] &= cand[w] - 1; }
                    if (!__any_sync(FULL, k >= 0)) break;
                    bool keep = false;
                    if (k >= 0) {
                        Atom av, aw, ax;
                        av.x = S.x[i]; av.y = S.y[i]; av.z = S.z[i]; av.r2 = S.r2[i];
                        aw.x = S.x[j]; aw.y = S.y[j]; aw.z = S.z[j]; aw.r2 = S.r2[j];
                        ax.x = S.x[k]; ax.y = S.y[k]; ax.z = S.z[k]; ax.r2 = S.r2[k];
                        const int ov = S.orig[i], ow = S.orig[j], ox = S.orig[k];
                        const Ortho e4 = ortho_tet(ou, au, ov, av, ow, aw, ox, ax, P.tol.eps_sing);   // pipeline.py:475-477
                        if (e4.singular)
                            record_singular(P, make_err_key(ST_TET, t, ((unsigned)tt << 8) | (unsigned)k), ou, ov, ow, ox, 4);
                        keep = e4.size <= P.tol.lim_a;                                               // pipeline.py:478
                    }
                    const unsigned m = __ballot_sync(FULL, keep);
                    const int cnt = __popc(m);
                    if (cnt) {
                        if (nqb + cnt > QBUF) flush_q();
                        if (keep) {
                            int slot = nqb + __popc(m & lanemask_lt());
                            S.qbuf_r[slot] = make_int4(t, S.rank[i], S.rank[j], S.rank[k]);
                            S.qbuf_l[slot] = i | (j << 8) | (k << 16);
                        }
                        nqb += cnt;
                        __syncwarp();
                    }
                }
            }
            __syncwarp();
        }
    }
    flush_t();
    flush_q();
    (void)warp;
}

}  // namespace axb
