// estimate.cuh -- stage one, potential edges (reference pipeline.py:316-359),
// one warp per generator ball; shared parameter block of the estimation kernels.
//
// A generator is the minimum-RANK vertex of a simplex (pipeline.py:10-15).
//   k_edges : scans the upper half of the generator's 5x5x5 cell block -- 13 rows
//             of cells, each a contiguous rank range -- lanes over candidates
//             (coalesced 32-byte atom loads), reach pre-filter + ortho-size test,
//             warp-ballot/popc compaction into the generator's partner list
//             (ascending rank).  Partner lists are staged in warp-private shared
//             memory and flushed with ONE global atomicAdd per ~32 generators.
// Potential triangles and tets: estimate2.cuh.
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
    int cull;                        // k_tri_tet2: drop / flag simplices dominated by a partner of their generator
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
// Two generators per warp pass: each 16-lane half sets up the candidate rows of one generator, the
// candidates of both are numbered consecutively and all 32 lanes then work through them together
// (a generator has ~15-35 candidates, so one generator alone leaves a warp half empty).
struct GenSlot {            // what a candidate lane needs to know about its generator
    double x, y, z, r2, reach;
    int orig, pad;
};

__global__ void __launch_bounds__(EST_WARPS * 32, 4) k_edges(EstParams P, int rank_lo, int rank_hi) {
    __shared__ int s_buf[EST_WARPS][EBUF];
    __shared__ int s_side[EST_WARPS][MAXP];                   // partners of the second generator of a pass
    __shared__ int s_gen[EST_WARPS][EGEN];
    __shared__ int s_goff[EST_WARPS][EGEN + 1];
    __shared__ int s_rs[EST_WARPS][32];                       // per row lane: first rank
    __shared__ int s_rp[EST_WARPS][32];                       // per row lane: first candidate number
    __shared__ int s_re[EST_WARPS][32];                       // per row lane: one past its last candidate number
    __shared__ GenSlot s_g[EST_WARPS][2];
    __shared__ unsigned char s_rowof[EST_WARPS][ROWOF_CAP];   // candidate number -> row lane (stamped)
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int half = lane >> 4, hl = lane & 15;
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
        for (int t0 = rank_lo + tile * EST_TILE + 2 * warp; t0 < t_end; t0 += 2 * EST_WARPS) {
            const int t = t0 + half;                        // this half's generator
            double ru = -1.0;
            if (t < t_end) ru = __ldg(P.reach + t);
            // the 13 rows of the 5x5x5 block whose balls can out-rank t (pipeline.py:332-338), each
            // trimmed to the cells a partner can sit in: a candidate v passes the reach filter only if
            // |v - u| <= reach_u + reach_v <= reach_u + reach_max, so cells whose nearest point is farther
            // than that from u (1e-9 slack, far above rounding) hold no partner.  Exact.
            int rs = 0, rc = 0;
            if (ru >= 0.0) {                                // viable generator (pipeline.py:336-337)
                const Atom au = load_atom(P.atoms, t);
                if (hl == 0) {
                    GenSlot &gs = s_g[warp][half];
                    gs.x = au.x; gs.y = au.y; gs.z = au.z; gs.r2 = au.r2; gs.reach = ru;
                    gs.orig = __ldg(P.orig + t);
                }
                if (hl < 13) {
                    const int4 cell = __ldg(P.cell_of_rank + t);
                    const int cx = cell.x, cy = cell.y, cz = cell.z;
                    int oy, oz;
                    if (hl < 3) { oy = hl; oz = 0; }
                    else { int q = hl - 3; oz = 1 + q / 5; oy = q % 5 - 2; }
                    const int y = cy + oy, z = cz + oz;
                    if (y >= 0 && y < g.dy && z < g.dz) {
                        const double R = ru + P.tol.reach_max;
                        const double R2 = R * R * (1.0 + 1e-9) + 1e-9;
                        const double xa = g.ox + (double)cx * g.side, ya = g.oy + (double)cy * g.side;
                        const double za = g.oz + (double)(cz + g.z_lo) * g.side;
                        const double dxl = fmax(au.x - xa, 0.0), dxh = fmax(xa + g.side - au.x, 0.0);
                        const double dyl = fmax(au.y - ya, 0.0), dyh = fmax(ya + g.side - au.y, 0.0);
                        const double dzh = fmax(za + g.side - au.z, 0.0);
                        const double gy = oy == 0 ? 0.0 : (oy > 0 ? dyh + (double)(oy - 1) * g.side : dyl + (double)(-oy - 1) * g.side);
                        const double gz = oz == 0 ? 0.0 : dzh + (double)(oz - 1) * g.side;
                        const double rem = R2 - gy * gy - gz * gz;
                        if (rem >= 0.0) {
                            int nl = 0, nh = 0;
                            if (dxl * dxl <= rem) { nl = 1; if ((dxl + g.side) * (dxl + g.side) <= rem) nl = 2; }
                            if (dxh * dxh <= rem) { nh = 1; if ((dxh + g.side) * (dxh + g.side) <= rem) nh = 2; }
                            const int x0 = max(cx - nl, 0), x1 = min(cx + nh, g.dx - 1);
                            int s, e;
                            row_range(g, x0, x1, y, z, s, e);
                            if (hl == 0) s = t + 1;         // own row: only ranks above t
                            rs = s;
                            rc = max(e - s, 0);
                        }
                    }
                }
            }
            int incl = rc;                                  // inclusive scan inside each half
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int v = __shfl_up_sync(FULL, incl, o, 16);
                if (hl >= o) incl += v;
            }
            const int tot_a = __shfl_sync(FULL, incl, 15), tot_b = __shfl_sync(FULL, incl, 31);
            const int total = tot_a + tot_b;
            if (total == 0) continue;
            if (nbuf + min(tot_a, MAXP) + min(tot_b, MAXP) > EBUF || ngen + 2 > EGEN) flush();
            __syncwarp();
            const int pre = incl - rc + (half ? tot_a : 0);
            s_rs[warp][lane] = rs; s_rp[warp][lane] = pre; s_re[warp][lane] = pre + rc;
            {
                const int pe = min(pre + rc, ROWOF_CAP);
                for (int p = pre; p < pe; ++p) s_rowof[warp][p] = (unsigned char)lane;
            }
            __syncwarp();
            int deg_a = 0, deg_b = 0;
            for (int p0 = 0; p0 < total; p0 += 32) {
                const int p = p0 + lane;
                bool keep = false;
                int cand = -1, sel = 0;
                if (p < total) {
                    int r = 0;
                    if (p < ROWOF_CAP) {
                        r = s_rowof[warp][p];
                    } else {
                        for (int k = 0; k < 32; ++k)
                            if (s_rp[warp][k] <= p && p < s_re[warp][k]) r = k;
                    }
                    sel = r >> 4;
                    cand = s_rs[warp][r] + (p - s_rp[warp][r]);
                    const double rv = __ldg(P.reach + cand);
                    const Atom av = load_atom(P.atoms, cand);
                    const GenSlot &gs = s_g[warp][sel];
                    Atom au;
                    au.x = gs.x; au.y = gs.y; au.z = gs.z; au.r2 = gs.r2;
                    if (rv >= 0.0 && reach_pair(av, rv, au, gs.reach)) {       // pipeline.py:341-344
                        const int ov = __ldg(P.orig + cand);
                        const Ortho o = ortho_edge(gs.orig, au, ov, av, P.tol.eps_sing);   // pipeline.py:355-356
                        if (o.singular)
                            record_singular(P, make_err_key(ST_EDGE, t0 + sel, (unsigned)(p - (sel ? tot_a : 0))), gs.orig, ov, -1, -1, 2);
                        keep = o.size <= P.tol.lim_a;                          // pipeline.py:358
                    }
                }
                const unsigned m = __ballot_sync(FULL, keep);
                const unsigned mb = __ballot_sync(FULL, keep && sel);
                const unsigned ma = m & ~mb;
                if (keep) {
                    if (sel) {
                        const int slot = deg_b + __popc(mb & lanemask_lt());
                        if (slot < MAXP) s_side[warp][slot] = cand;
                    } else {
                        const int slot = deg_a + __popc(ma & lanemask_lt());
                        if (slot < MAXP) s_buf[warp][nbuf + slot] = cand;
                    }
                }
                deg_a += __popc(ma);
                deg_b += __popc(mb);
            }
            if (deg_a > MAXP || deg_b > MAXP) {
                if (lane == 0) atomicOr(&P.ctr->overflow, 1u);                 // AXB_ERR_DENSITY
                deg_a = min(deg_a, MAXP);
                deg_b = min(deg_b, MAXP);
            }
            __syncwarp();
            if (deg_a > 0) {
                if (lane == 0) { s_gen[warp][ngen] = t0; s_goff[warp][ngen] = nbuf; }
                nbuf += deg_a;
                ngen += 1;
                max_deg = max(max_deg, (unsigned)deg_a);
                pairs += (unsigned long long)deg_a * (unsigned)(deg_a - 1) / 2;
            }
            if (deg_b > 0) {
                for (int i = lane; i < deg_b; i += 32) s_buf[warp][nbuf + i] = s_side[warp][i];
                if (lane == 0) { s_gen[warp][ngen] = t0 + 1; s_goff[warp][ngen] = nbuf; }
                nbuf += deg_b;
                ngen += 1;
                max_deg = max(max_deg, (unsigned)deg_b);
                pairs += (unsigned long long)deg_b * (unsigned)(deg_b - 1) / 2;
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

__device__ __forceinline__ int nth_set_bit(unsigned long long m, int n) {
    for (int q = 0; q < n; ++q) m &= m - 1;
    return __ffsll((long long)m) - 1;
}

}  // namespace axb
