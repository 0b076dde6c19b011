// estimate.cuh -- stage one, potential edges (reference pipeline.py:316-359),
// one warp per generator ball; shared parameter block of the estimation kernels.
//
// A generator is the minimum-RANK vertex of a simplex (pipeline.py:10-15).
//   k_edges : a warp takes batches of 8 consecutive generators; the upper half of each
//             generator's 5x5x5 cell block is 13 rows of cells, each a contiguous rank
//             range; the batch's candidates are flattened so lanes stay packed
//             (one 32-byte load per candidate), reach pre-filter, queued ortho-size
//             tests, warp-ballot/popc compaction into the partner lists (ascending
//             rank).  Lists are staged in warp-private shared memory and flushed with
//             ONE global atomicAdd per ~32 generators.
// Potential triangles and tets: estimate3.cuh.
#pragma once

#include "common.cuh"
#include "predicates.cuh"

namespace axb {

constexpr int EST_WARPS = 8;
#ifndef EBUF_V
#define EBUF_V 320
#endif
constexpr int EBUF = EBUF_V;   // partner ranks staged per warp
constexpr int EGEN = 32;       // generators staged per warp
constexpr int MAXP = 256;      // AXB_MAX_PARTNERS

struct EstParams {
    GridView g;
    Tol tol;
    const Atom *atoms;
    const Atom *xyzr;           // (x, y, z, reach) per rank
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
    int cull;                        // k_tri_tet3: drop / flag simplices dominated by a partner of their generator
    int err_rank_hi;                 // singular solves are reported for generators below this rank only (slab: the
                                     // upper halo's enumeration is incomplete; its owner reports it)
    int own_lo;                      // slab: first owned rank; a lower-halo generator matters only if a partner reaches it
};

__device__ __forceinline__ void sort_small(int *v, int k) {
    for (int a = 1; a < k; ++a) {
        int x = v[a], b = a - 1;
        while (b >= 0 && v[b] > x) { v[b + 1] = v[b]; --b; }
        v[b + 1] = x;
    }
}

// (takes what it needs BY VALUE: a reference to the kernel's parameter block would force a copy of the whole
// block into a local-memory stack frame)
__device__ __noinline__ void record_singular_impl(Counters *ctr, ErrRecord *errs, unsigned long long report_key,
                                                  unsigned long long key, int v0, int v1, int v2, int v3, int nv) {
    atomicMin(&ctr->err_key, key);
    ErrRecord r;
    r.key = key;
    r.verts[0] = v0; r.verts[1] = v1; r.verts[2] = v2; r.verts[3] = v3;
    sort_small(r.verts, nv);
    r.nverts = nv;
    r.pad = 0;
    if (report_key) {
        if (key == report_key) errs[0] = r;
    } else {
        unsigned slot = atomicAdd(&ctr->err_count, 1u);
        if (slot < ERR_CAP) errs[slot] = r;
    }
}

__device__ __forceinline__ void record_singular(const EstParams &P, unsigned long long key, int v0, int v1, int v2, int v3,
                                                int nv) {
    record_singular_impl(P.ctr, P.errs, P.report_key, key, v0, v1, v2, v3, nv);
}

// ---------------------------------------------------------------- k_edges
// A warp takes a BATCH of up to 8 consecutive generators and runs every phase over the batch's
// flattened work so lanes stay packed (one generator alone has ~33 candidates, ~5 partners):
//   A  the 8 x 13 candidate rows (one lane per row, exact geometric trimming) -> (first rank, count),
//      warp scan -> candidate numbering, stamped candidate -> row table
//   B  dense over the candidates: ONE 32-byte (x, y, z, reach) load each, reach pre-filter
//      (pipeline.py:341-344), passing pairs appended to a warp queue with ballot/popc
//   C  dense over the queue: ortho2 + size test (pipeline.py:355-358), kept pairs compacted in place;
//      the queue is generator-major and rank-ascending, so what is left IS the concatenation of the
//      partner lists (pipeline.py:362-370)
// Partner lists are staged in warp-private shared memory and flushed with one global atomicAdd per
// ~32 generators.
struct __align__(16) GenSlot {   // what a candidate lane needs to know about its generator
    double x, y, z, reach;       // two 16-byte shared loads feed the reach pre-filter
    double r2;
    int orig, pad;
};

// Per-generator trimming table (computed once by one lane): a candidate v passes the reach filter only if
// |v - u| <= reach_u + reach_v <= reach_u + reach_max =: R, so cells whose nearest point is farther than
// R from u (1e-9 slack, far above rounding) hold no partner.  rem = (R2 - gy2[oy + 2]) - gz2[oz] is what is
// left for the x direction in row (oy, oz); the row spans cells cx - nl .. cx + nh with nl / nh = how many of
// xl[0..1] / xh[0..1] (squared distances to the near faces of the neighbouring columns) fit into rem.
struct __align__(16) GenGeo {
    double xl[2], xh[2];
    double R2, gz2[3];
    double gy2[5];
    int cx, cy, cz;
};

#ifndef E2_GB_V
#define E2_GB_V 8
#endif
constexpr int E2_GB = E2_GB_V;                // generators per warp batch
constexpr int E2_ROWS = 13;                   // rows of the 5x5x5 block that can out-rank the generator
constexpr int E2_ITEMS = E2_GB * E2_ROWS;     // 104 row items, 4 rounds of 32 lanes
#ifndef E2_CCAP_V
#define E2_CCAP_V 512
#endif
#ifndef E2_QCAP_V
#define E2_QCAP_V 320
#endif
constexpr int E2_CCAP = E2_CCAP_V;                  // candidates of a batch covered by the stamped row table
constexpr int E2_QCAP = E2_QCAP_V;                  // queued pairs per warp (> MAXP + 32)
#ifndef E2_MINB
#define E2_MINB 4
#endif

struct E2Warp {
    GenSlot g[E2_GB];
    GenGeo geo[E2_GB];
    int2 row_info[E2_ITEMS];                  // (first rank - first candidate number, generator slot)
    int row_pre[E2_ITEMS + 1];
    int q_cand[E2_QCAP];
    unsigned short q_ord[E2_QCAP];            // candidate number inside the batch (error key only)
    unsigned char q_gen[E2_QCAP];
    unsigned char rowof[E2_CCAP];
    int buf[EBUF];
    int gen[EGEN];
    int goff[EGEN + 1];
    int first[E2_GB], last[E2_GB];
};

__global__ void __launch_bounds__(EST_WARPS * 32, E2_MINB) k_edges(EstParams P, int rank_lo, int rank_hi) {
    extern __shared__ __align__(16) unsigned char s_raw_e2[];      // EST_WARPS x E2Warp (54 KB: dynamic)
    const int warp = threadIdx.x >> 5, lane = lane_id();
    E2Warp &S = reinterpret_cast<E2Warp *>(s_raw_e2)[warp];
    const GridView &g = P.g;
    int nbuf = 0, ngen = 0;                 // warp-uniform staging state
    unsigned max_deg = 0;                   // lane-local, reduced at the end
    unsigned long long pairs = 0;

    auto flush = [&]() {
        if (ngen == 0) return;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&P.ctr->n_pe, (unsigned)nbuf);
        base = __shfl_sync(FULL, base, 0);
        if ((unsigned long long)base + (unsigned)nbuf <= P.pe_cap) {
            if (lane == 0) S.goff[ngen] = nbuf;
            __syncwarp();
            if (lane < ngen) {
                int t = S.gen[lane];
                P.adj_off[t] = base + (unsigned)S.goff[lane];
                P.deg[t] = S.goff[lane + 1] - S.goff[lane];
            }
            for (int idx = lane; idx < nbuf; idx += 32) {
                int gi = 0;                                 // last staged generator with goff <= idx
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (gi + step < ngen && S.goff[gi + step] <= idx) gi += step;
                P.pe_v[base + idx] = S.buf[idx];
                P.pe_u[base + idx] = S.gen[gi];
            }
        } else if (lane == 0) {
            atomicOr(&P.ctr->overflow, 1u << 4);           // potential-edge buffer too small: caller re-runs
        }
        __syncwarp();
        nbuf = 0;
        ngen = 0;
    };

    const int nbatch = (rank_hi - rank_lo + E2_GB - 1) / E2_GB;
    for (int b = blockIdx.x * EST_WARPS + warp; b < nbatch; b += gridDim.x * EST_WARPS) {
        const int tb = rank_lo + b * E2_GB;
        const int tb_end = min(tb + E2_GB, rank_hi);
        int ts = tb, gb = E2_GB;
        while (ts < tb_end) {
            gb = min(gb, tb_end - ts);                      // generators offered to this pass
            // ---- A: candidate rows.  The 13 rows of the 5x5x5 block whose balls can out-rank t
            // (pipeline.py:332-338), each trimmed to the cells a partner can sit in: a candidate v passes the
            // reach filter only if |v - u| <= reach_u + reach_v <= reach_u + reach_max, so cells whose nearest
            // point is farther than that from u (1e-9 slack, far above rounding) hold no partner.  Exact.
            // A0: one lane per generator loads its record and fills the trimming table
            if (lane < E2_GB) {
                GenSlot &q = S.g[lane];
                double ru = -1.0;
                if (lane < gb) ru = __ldg(P.reach + ts + lane);
                q.reach = ru;
                if (ru >= 0.0) {                            // viable generator (pipeline.py:336-337)
                    const int t = ts + lane;
                    const Atom au = load_atom(P.atoms, t);
                    const int4 cell = __ldg(P.cell_of_rank + t);
                    q.x = au.x; q.y = au.y; q.z = au.z; q.r2 = au.r2;
                    q.orig = __ldg(P.orig + t);
                    GenGeo &G = S.geo[lane];
                    const double R = ru + P.tol.reach_max;
                    G.R2 = R * R * (1.0 + 1e-9) + 1e-9;
                    const double xa = g.ox + (double)cell.x * g.side, ya = g.oy + (double)cell.y * g.side;
                    const double za = g.oz + (double)(cell.z + g.z_lo) * g.side;
                    const double dxl = fmax(au.x - xa, 0.0), dxh = fmax(xa + g.side - au.x, 0.0);
                    const double dyl = fmax(au.y - ya, 0.0), dyh = fmax(ya + g.side - au.y, 0.0);
                    const double dzh = fmax(za + g.side - au.z, 0.0);
                    G.xl[0] = dxl * dxl; G.xl[1] = (dxl + g.side) * (dxl + g.side);
                    G.xh[0] = dxh * dxh; G.xh[1] = (dxh + g.side) * (dxh + g.side);
                    G.gy2[0] = (dyl + g.side) * (dyl + g.side); G.gy2[1] = dyl * dyl; G.gy2[2] = 0.0;
                    G.gy2[3] = dyh * dyh; G.gy2[4] = (dyh + g.side) * (dyh + g.side);
                    G.gz2[0] = 0.0; G.gz2[1] = dzh * dzh; G.gz2[2] = (dzh + g.side) * (dzh + g.side);
                    G.cx = cell.x; G.cy = cell.y; G.cz = cell.z;
                }
            }
            __syncwarp();
            // A1: one lane per row; the row-bound loads of all four rounds are independent of each other
            int rs[(E2_ITEMS + 31) / 32], rc[(E2_ITEMS + 31) / 32];
#pragma unroll
            for (int r4 = 0; r4 < (E2_ITEMS + 31) / 32; ++r4) {
                const int item = r4 * 32 + lane;
                const int gs = min(item / E2_ROWS, E2_GB - 1), hl = item - gs * E2_ROWS;
                rs[r4] = 0; rc[r4] = 0;
                bool ok = item < E2_ITEMS && S.g[gs].reach >= 0.0;
                const GenGeo &G = S.geo[gs];
                int oy, oz;
                if (hl < 3) { oy = hl; oz = 0; }
                else { const int q = hl - 3; oz = 1 + q / 5; oy = q % 5 - 2; }
                int x0 = 0, x1 = 0, y = 0, z = 0;
                if (ok) {
                    y = G.cy + oy; z = G.cz + oz;
                    const double rem = (G.R2 - G.gy2[oy + 2]) - G.gz2[oz];
                    ok = y >= 0 && y < g.dy && z < g.dz && rem >= 0.0;
                    const int nl = (G.xl[0] <= rem) + (G.xl[1] <= rem), nh = (G.xh[0] <= rem) + (G.xh[1] <= rem);
                    x0 = max(G.cx - nl, 0); x1 = min(G.cx + nh, g.dx - 1);
                }
                if (g.cell_start) {                         // dense table: clamped addresses, no branch around the loads
                    const int row = ok ? g.dx * (y + g.dy * z) : 0;
                    const int s = (int)__ldg(g.cell_start + (ok ? row + x0 : 0));
                    const int e = (int)__ldg(g.cell_start + (ok ? row + x1 + 1 : 0));
                    rs[r4] = s; rc[r4] = e - s;
                } else if (ok) {
                    int s, e;
                    row_range(g, x0, x1, y, z, s, e);
                    rs[r4] = s; rc[r4] = e - s;
                }
                if (ok && hl == 0) { rc[r4] -= (ts + gs + 1) - rs[r4]; rs[r4] = ts + gs + 1; }   // own row: only ranks above t
                rc[r4] = ok ? max(rc[r4], 0) : 0;
            }
            int carry = 0;
#pragma unroll
            for (int r4 = 0; r4 < (E2_ITEMS + 31) / 32; ++r4) {
                const int item = r4 * 32 + lane;
                const int incl = warp_incl_scan(rc[r4]);
                if (item < E2_ITEMS) {
                    const int pre = carry + incl - rc[r4];
                    S.row_pre[item] = pre;
                    S.row_info[item] = make_int2(rs[r4] - pre, item / E2_ROWS);
                }
                carry += __shfl_sync(FULL, incl, 31);
            }
            if (lane == 0) S.row_pre[E2_ITEMS] = carry;
            __syncwarp();
            // as many generators as the stamped table covers (at least one)
            int gu = gb;
            while (gu > 1 && S.row_pre[gu * E2_ROWS] > E2_CCAP) --gu;
            const int total = S.row_pre[gu * E2_ROWS];
            if (total > 0) {
#pragma unroll
                for (int r4 = 0; r4 < (E2_ITEMS + 31) / 32; ++r4) {
                    const int item = r4 * 32 + lane;
                    if (item < gu * E2_ROWS) {
                        const int pb = S.row_pre[item], pe = min(S.row_pre[item + 1], E2_CCAP);
                        for (int p = pb; p < pe; ++p) S.rowof[p] = (unsigned char)item;
                    }
                }
                __syncwarp();
                int qn = 0, solved = 0;                     // warp-uniform: queue fill, settled prefix
                // ---- C (defined first): ortho2 over the unsettled part of the queue, kept pairs compacted in place
                auto settle = [&]() {
                    int w = solved;
                    for (int x0 = solved; x0 < qn; x0 += 32) {
                        const int x = x0 + lane;
                        bool keep = false;
                        int cand = 0, gs = 0, ord = 0;
                        if (x < qn) {
                            cand = S.q_cand[x]; gs = S.q_gen[x]; ord = S.q_ord[x];
                            const GenSlot &q = S.g[gs];
                            Atom au;
                            au.x = q.x; au.y = q.y; au.z = q.z; au.r2 = q.r2;
                            const Atom av = load_atom(P.atoms, cand);
                            const int ov = __ldg(P.orig + cand);
                            const Ortho o = ortho_edge(q.orig, au, ov, av, P.tol.eps_sing);        // pipeline.py:355-356
                            if (o.singular && ts + gs < P.err_rank_hi)   // ordinal = candidate number inside its generator
                                record_singular(P, make_err_key(ST_EDGE, ts + gs, (unsigned)(ord - S.row_pre[gs * E2_ROWS])), q.orig, ov, -1, -1, 2);
                            keep = o.size <= P.tol.lim_a;                                          // pipeline.py:358
                        }
                        const unsigned m = __ballot_sync(FULL, keep);
                        __syncwarp();                       // every lane has read its entry before the prefix is overwritten
                        if (keep) {
                            const int pos = w + __popc(m & lanemask_lt());
                            S.q_cand[pos] = cand; S.q_gen[pos] = (unsigned char)gs;
                        }
                        w += __popc(m);
                        __syncwarp();
                    }
                    qn = w;
                    solved = w;
                };
                // ---- B: reach pre-filter over the flattened candidates
                auto lookup = [&](int p, int &cand, int &gs) {
                    int item;
                    if (p < E2_CCAP) {
                        item = S.rowof[p];
                    } else {                                // one very dense generator: search its 13 rows
                        item = 0;
                        for (int k = 1; k < E2_ROWS; ++k)
                            if (S.row_pre[k] <= p) item = k;
                    }
                    const int2 info = S.row_info[item];
                    gs = info.y;
                    cand = p + info.x;
                };
                bool crowded = false;                       // the batch has more partners than the queue holds
                int cand_n = 0, gs_n = 0;
                if (lane < total) {
                    lookup(lane, cand_n, gs_n);
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + cand_n));
                }
                for (int p0 = 0; p0 < total; p0 += 32) {
                    const int p = p0 + lane;
                    const int cand = cand_n, gs = gs_n;
                    // the record of the NEXT round is requested (L1 prefetch, no destination register) before this
                    // round's is loaded and tested
                    if (p + 32 < total) {
                        lookup(p + 32, cand_n, gs_n);
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + cand_n));
                    }
                    Atom av;
                    av.x = av.y = av.z = 0.0; av.r2 = -1.0;
                    if (p < total) av = load_atom(P.xyzr, cand);            // (x, y, z, reach)
                    bool pass = false;
                    if (p < total) {
                        const GenSlot &q = S.g[gs];
                        const double dx = av.x - q.x, dy = av.y - q.y, dz = av.z - q.z;
                        const double lims = av.r2 + q.reach;
                        pass = av.r2 >= 0.0 && (dx * dx + dy * dy) + dz * dz <= lims * lims;   // pipeline.py:341-344
                    }
                    const unsigned m = __ballot_sync(FULL, pass);
                    if (m) {
                        if (qn + 32 > E2_QCAP) {
                            settle();
                            if (qn + 32 > E2_QCAP) { crowded = true; break; }
                        }
                        if (pass) {
                            const int pos = qn + __popc(m & lanemask_lt());
                            S.q_cand[pos] = cand; S.q_gen[pos] = (unsigned char)gs; S.q_ord[pos] = (unsigned short)min(p, 65535);
                        }
                        qn += __popc(m);
                        __syncwarp();
                    }
                }
                if (crowded) {
                    // more than E2_QCAP - 32 >= AXB_MAX_PARTNERS kept pairs: halve the batch and redo it; for a
                    // single generator it is the density limit (AXB_ERR_DENSITY)
                    if (gu > 1) { gb = gu / 2; continue; }
                    if (lane == 0) atomicOr(&P.ctr->overflow, 1u);
                    qn = 0; solved = 0;
                }
                settle();
                // ---- partner lists: the queue is generator-major, so list boundaries are where q_gen changes
                if (lane < E2_GB) { S.first[lane] = 0; S.last[lane] = 0; }
                __syncwarp();
                for (int x = lane; x < qn; x += 32) {
                    const int gs = S.q_gen[x];
                    if (x == 0 || S.q_gen[x - 1] != gs) S.first[gs] = x;
                    if (x == qn - 1 || S.q_gen[x + 1] != gs) S.last[gs] = x + 1;
                }
                __syncwarp();
                if (qn > 0) {
                    if (nbuf + qn > EBUF || ngen + gu > EGEN) flush();
                    int d = 0, f = 0;
                    if (lane < gu) { f = S.first[lane]; d = S.last[lane] - f; }
                    if (d > MAXP) atomicOr(&P.ctr->overflow, 1u);              // AXB_ERR_DENSITY
                    const unsigned mg = __ballot_sync(FULL, d > 0);
                    if (d > 0) {
                        const int slot = ngen + __popc(mg & lanemask_lt());
                        S.gen[slot] = ts + lane;
                        S.goff[slot] = nbuf + f;
                        max_deg = max(max_deg, (unsigned)d);
                        pairs += (unsigned long long)d * (unsigned)(d - 1) / 2;
                    }
                    for (int x = lane; x < qn; x += 32) S.buf[nbuf + x] = S.q_cand[x];
                    ngen += __popc(mg);
                    nbuf += qn;
                    __syncwarp();
                }
            }
            ts += gu;
            gb = E2_GB;
        }
    }
    flush();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        max_deg = max(max_deg, __shfl_xor_sync(FULL, max_deg, o));
        pairs += __shfl_xor_sync(FULL, pairs, o);
    }
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
