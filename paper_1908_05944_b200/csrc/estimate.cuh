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
                    int x0 = max(cx - 2, 0), x1 = min(cx + 2, g.dx - 1);
                    int s, e;
                    row_range(g, x0, x1, y, z, s, e);
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

__device__ __forceinline__ int nth_set_bit(unsigned long long m, int n) {
    for (int q = 0; q < n; ++q) m &= m - 1;
    return __ffsll((long long)m) - 1;
}

}  // namespace axb
