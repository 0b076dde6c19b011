// edges.cuh -- stage one, potential edges (reference pipeline.py:316-359): k_edges.
//
// A generator is the minimum-RANK vertex of a simplex (pipeline.py:10-15); its candidate partners are the
// balls of the 13 cell rows of its 5x5x5 block that can out-rank it (pipeline.py:332-338), each row one
// contiguous rank range.
//
// Lane = generator.  A warp owns a tile of 32 consecutive generators; every lane keeps ITS generator's
// record in registers, so the per-candidate work -- one 32-byte (x, y, z, reach) load and the reach
// pre-filter (pipeline.py:341-344) -- touches no shared memory at all, and neighbouring lanes (neighbouring
// cells) read overlapping rank ranges, which the L1 serves as broadcasts.  (The predecessor flattened
// (generator, candidate) pairs over the lanes: perfectly packed, but every candidate then paid four shared
// look-ups to find its generator, and the kernel ran at 78 % of the L1/shared data pipe with 16 M bank
// conflicts per million balls -- ncu r2a.)
//   A  every lane trims its 13 rows exactly (a partner must lie within reach_u + reach_max of u, so cells
//      whose nearest point is farther hold none), fetches the 26 row bounds back to back, and parks the
//      non-empty rows in its column of a [13][32] shared table;
//   B  every lane walks its own rows as one flattened sequence; pairs that pass the pre-filter are queued
//      with ballot/popc (warp-wide queue in shared memory);
//   C  dense over the queue: ortho2 + size test (pipeline.py:355-358), kept pairs compacted in place;
//   D  stable counting sort of the kept pairs by generator (every generator's pairs were queued in
//      ascending rank, so its partner list comes out ascending = pipeline.py:362-370), one global
//      atomicAdd per tile, coalesced list stores.
#pragma once

#include "common.cuh"
#include "estimate.cuh"
#include "predicates.cuh"

namespace axb {

#ifndef EL_WARPS_V
#define EL_WARPS_V 4
#endif
#ifndef EL_MINB_V
#define EL_MINB_V 7
#endif
#ifndef EL_QCAP_V
#define EL_QCAP_V 512
#endif
constexpr int EL_WARPS = EL_WARPS_V;        // warps per block (each one independent)
constexpr int EL_MINB = EL_MINB_V;          // resident blocks per SM the registers must allow
constexpr int EL_QCAP = EL_QCAP_V;          // queued pairs per warp (> AXB_MAX_PARTNERS + 32)
constexpr int EL_ROWS = 13;
#ifndef EL_PREF_ROW
#define EL_PREF_ROW 0
#endif
#ifndef EL_PREF_AHEAD
#define EL_PREF_AHEAD 1
#endif
#ifndef EL_PREF_TILE
#define EL_PREF_TILE 1
#endif
#ifndef EL_WALK2
#define EL_WALK2 3           // candidates per lane and walk iteration (0: the one-at-a-time loop)
#endif
#ifndef EL_BUDGET_V
#define EL_BUDGET_V 2400
#endif
constexpr int EL_BUDGET = EL_BUDGET_V;      // candidates a pass takes on (about a sixth of them end up in the queue)

struct __align__(16) ELWarp {
    union {
        int2 rows[EL_ROWS][32];             // A-C: [k][lane] = (first rank, end rank) of the lane's k-th non-empty row
        int sorted[EL_ROWS * 32 * 2];       // D: partner ranks grouped by generator
    } u;
    int q_cand[EL_QCAP];
    unsigned char q_gen[EL_QCAP];
    double gx[32], gy[32], gz[32], gr2[32]; // the tile's generators by lane (the dense phase C names them by slot)
    int gorig[32];
    int nrow[32];
    int cnt[32];
    int off[33];
};
static_assert(EL_ROWS * 32 * 2 >= EL_QCAP, "the sorted list aliases the row table");

// Phase A of k_edges for one lane: loads generator t (if `active`), publishes its record in the warp's slot table,
// trims its 13 candidate rows exactly and parks the non-empty ones in the lane's column of S.u.rows.
// Returns the number of parked rows; ux, uy, uz, ureach = the generator (ureach < 0: not viable / idle lane).
__device__ __forceinline__ int lane_rows(const EstParams &P, ELWarp &S, int t, int lane, bool active, double &ux, double &uy,
                                         double &uz, double &ureach) {
    const GridView &g = P.g;
    int nr = 0;
    if (active) ureach = __ldg(P.reach + t);
    if (ureach >= 0.0) {                            // viable generator (pipeline.py:336-337)
        const Atom au = load_atom(P.atoms, t);
        const int4 cell = __ldg(P.cell_of_rank + t);
        ux = au.x; uy = au.y; uz = au.z;
        S.gx[lane] = au.x; S.gy[lane] = au.y; S.gz[lane] = au.z; S.gr2[lane] = au.r2;
        S.gorig[lane] = __ldg(P.orig + t);
        // trimming table: a candidate v passes the pre-filter only if |v - u| <= reach_u + reach_v <= reach_u +
        // reach_max =: R, so cells whose nearest point is farther than R from u (1e-9 slack, far above rounding)
        // hold no partner.  rem = (R2 - gy2) - gz2 is what is left for the x direction in row (oy, oz).
        const double R = ureach + P.tol.reach_max;
        const double R2 = R * R * (1.0 + 1e-9) + 1e-9;
        const double xa = g.ox + (double)cell.x * g.side, ya = g.oy + (double)cell.y * g.side;
        const double za = g.oz + (double)(cell.z + g.z_lo) * g.side;
        const double dxl = fmax(au.x - xa, 0.0), dxh = fmax(xa + g.side - au.x, 0.0);
        const double dyl = fmax(au.y - ya, 0.0), dyh = fmax(ya + g.side - au.y, 0.0);
        const double dzh = fmax(za + g.side - au.z, 0.0);
        const double xl0 = dxl * dxl, xl1 = (dxl + g.side) * (dxl + g.side);
        const double xh0 = dxh * dxh, xh1 = (dxh + g.side) * (dxh + g.side);
        const double gy2[5] = {(dyl + g.side) * (dyl + g.side), dyl * dyl, 0.0, dyh * dyh, (dyh + g.side) * (dyh + g.side)};
        const double gz2[3] = {0.0, dzh * dzh, (dzh + g.side) * (dzh + g.side)};
        int rs[EL_ROWS], re[EL_ROWS];
#pragma unroll
        for (int hl = 0; hl < EL_ROWS; ++hl) {      // rows in ascending key order: (oz 0: oy 0..2), (oz 1, 2: oy -2..2)
            const int oz = hl < 3 ? 0 : 1 + (hl - 3) / 5;
            const int oy = hl < 3 ? hl : (hl - 3) % 5 - 2;
            const int y = cell.y + oy, z = cell.z + oz;
            const double rem = (R2 - gy2[oy + 2]) - gz2[oz];
            const bool ok = y >= 0 && y < g.dy && z < g.dz && rem >= 0.0;
            const int nl = (xl0 <= rem) + (xl1 <= rem), nh = (xh0 <= rem) + (xh1 <= rem);
            const int x0 = max(cell.x - nl, 0), x1 = min(cell.x + nh, g.dx - 1);
            int s = 0, e = 0;
            if (g.cell_start) {                     // dense table: clamped addresses, all 26 loads in flight together
                const int row = ok ? g.dx * (y + g.dy * z) : 0;
                s = (int)__ldg(g.cell_start + (ok ? row + x0 : 0));
                e = (int)__ldg(g.cell_start + (ok ? row + x1 + 1 : 0));
            } else if (ok) {
                row_range(g, x0, x1, y, z, s, e);
            }
            if (hl == 0) s = max(s, t + 1);         // own row: only ranks above t
            rs[hl] = s;
            re[hl] = ok ? e : s;
        }
#pragma unroll
        for (int hl = 0; hl < EL_ROWS; ++hl)
            if (re[hl] > rs[hl]) { S.u.rows[nr][lane] = make_int2(rs[hl], re[hl]); ++nr; }
    }
    return nr;
}

// One generator with more partners than the pair queue holds (large alpha: hundreds of partners): k_edges marks it
// (deg = -1) and k_edges_heavy, launched only when the counters say there is one, takes it.  The warp sweeps
// its candidate rows twice, 32 candidates per round in rank order: the first sweep counts the kept pairs, one
// atomicAdd reserves the list, the second sweep writes it (ballot/popc keeps the ascending order).  Generator 0 of
// the pass: its record is in S.g*[0], its rows in S.u.rows[.][0].  Returns the number of partners.
__device__ __forceinline__ unsigned heavy_generator(const EstParams &P, ELWarp &S, int t, int lane) {
    Atom au;
    au.x = S.gx[0]; au.y = S.gy[0]; au.z = S.gz[0]; au.r2 = S.gr2[0];
    const int ou = S.gorig[0];
    const double ureach = __ldg(P.reach + t);
    const int nr = S.nrow[0];
    unsigned total = 0, base = 0;
    for (int sweep = 0; sweep < 2; ++sweep) {
        unsigned w = 0, ord = 0;
        for (int k = 0; k < nr; ++k) {
            const int2 rw = S.u.rows[k][0];
            for (int p0 = rw.x; p0 < rw.y; p0 += 32) {
                const int p = p0 + lane;
                bool keep = false;
                if (p < rw.y) {
                    const Atom xr = load_atom(P.xyzr, p);
                    const double dx = xr.x - au.x, dy = xr.y - au.y, dz = xr.z - au.z;
                    const double lims = xr.r2 + ureach;
                    if (xr.r2 >= 0.0 && (dx * dx + dy * dy) + dz * dz <= lims * lims) {                 // pipeline.py:341-344
                        const Atom av = load_atom(P.atoms, p);
                        const int ov = __ldg(P.orig + p);
                        const Ortho o = ortho_edge(ou, au, ov, av, P.tol.eps_sing);                     // pipeline.py:355-356
                        if (sweep == 0 && o.singular && t < P.err_rank_hi)
                            record_singular(P, make_err_key(ST_EDGE, t, ord + (unsigned)(p - p0)), ou, ov, -1, -1, 2);
                        keep = o.size <= P.tol.lim_a;                                                   // pipeline.py:358
                    }
                }
                const unsigned m = __ballot_sync(FULL, keep);
                if (sweep == 1 && keep && (unsigned long long)base + total <= P.pe_cap) {
                    const unsigned at = base + w + (unsigned)__popc(m & lanemask_lt());
                    P.pe_v[at] = p;
                    P.pe_u[at] = t;
                }
                w += (unsigned)__popc(m);
                ord += (unsigned)min(32, rw.y - p0);
            }
        }
        if (sweep == 0) {
            total = w;
            if (lane == 0 && total) base = atomicAdd(&P.ctr->n_pe, total);
            base = __shfl_sync(FULL, base, 0);
            if ((unsigned long long)base + total > P.pe_cap) {
                if (lane == 0) atomicOr(&P.ctr->overflow, 1u << 4);   // potential-edge buffer too small: caller re-runs
            } else if (lane == 0 && total) {
                P.adj_off[t] = base;
                P.deg[t] = (int)total;
            }
        }
    }
    return total;
}

// dyn: tiles are claimed from a global counter (dense regions make them very unequal); with at most one tile per
// warp the plain assignment is used -- the claims of thousands of warps on one address would only cost time
__global__ void __launch_bounds__(EL_WARPS * 32, EL_MINB) k_edges(EstParams P, int rank_lo, int rank_hi, int dyn) {
    extern __shared__ __align__(16) unsigned char s_raw_el[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    ELWarp &S = reinterpret_cast<ELWarp *>(s_raw_el)[warp];
    unsigned max_deg = 0;
    unsigned long long pairs = 0;

    const int ntiles = (rank_hi - rank_lo + 31) / 32;
    // the claim for the NEXT tile is issued before the current one is processed, so its round trip is hidden
    int tile_n = blockIdx.x * EL_WARPS + warp;
    if (dyn && lane == 0) tile_n = (int)atomicAdd(&P.ctr->work_next[0], 1u);
    for (;;) {
        const int tile = __shfl_sync(FULL, tile_n, 0);
        if (tile >= ntiles) break;
        if (!dyn) tile_n = tile + gridDim.x * EL_WARPS;
        else if (lane == 0) tile_n = (int)atomicAdd(&P.ctr->work_next[0], 1u);
        const int tile_lo = rank_lo + tile * 32;
        const int tile_hi = min(tile_lo + 32, rank_hi);
        int ts = tile_lo, gb = 32;
        while (ts < tile_hi) {
            gb = min(gb, tile_hi - ts);                     // generators offered to this pass (lanes >= gb idle)
            const int t = ts + lane;
            // ---- A: the lane's generator and its candidate rows
            double ux = 0.0, uy = 0.0, uz = 0.0, ureach = -1.0;
            int nr = lane_rows(P, S, t, lane, lane < gb, ux, uy, uz, ureach);
            S.nrow[lane] = nr;
            __syncwarp();
            // a pass takes as many generators as fit the candidate budget (dense cores: three times the balls per cell):
            // the queue must hold every kept pair of the pass, and finding that out half-way costs the whole walk
            {
                int tot = 0;
                for (int k = 0; k < nr; ++k) { const int2 q = S.u.rows[k][lane]; tot += q.y - q.x; }
                const int incl = warp_incl_scan(tot);
                const int fit = __popc(__ballot_sync(FULL, incl <= EL_BUDGET));     // totals ascend: the set is a prefix
                if (fit < gb) {
                    gb = max(fit, 1);
                    if (lane >= gb) nr = 0;
                }
            }

#if EL_PREF_TILE
            {   // the next tile's generators (record, reach, cell) are requested now; phase A finds them in L1 / L2
                const int tnx = __shfl_sync(FULL, tile_n, 0);
                const int tq = rank_lo + tnx * 32 + lane;
                if (ts == tile_lo && tnx < ntiles && tq < rank_hi) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.atoms + tq));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.reach + tq));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.cell_of_rank + tq));
                }
            }
#endif
            int qn = 0, solved = 0;                         // warp-uniform: queue fill, settled prefix
            // ---- C (defined first): ortho2 over the unsettled part of the queue, kept pairs compacted in place
            auto settle = [&]() {
                int w = solved;
                for (int x0 = solved; x0 < qn; x0 += 32) {
                    const int x = x0 + lane;
                    bool keep = false;
                    int cand = 0, gs = 0;
                    if (x < qn) {
                        cand = S.q_cand[x]; gs = S.q_gen[x];
                        Atom au;
                        au.x = S.gx[gs]; au.y = S.gy[gs]; au.z = S.gz[gs]; au.r2 = S.gr2[gs];
                        const int ou = S.gorig[gs];
                        const Atom av = load_atom(P.atoms, cand);
                        const int ov = __ldg(P.orig + cand);
                        const Ortho o = ortho_edge(ou, au, ov, av, P.tol.eps_sing);            // pipeline.py:355-356
                        if (o.singular && ts + gs < P.err_rank_hi) {
                            // ordinal = candidate number inside its generator's enumeration (rows are disjoint, ascending)
                            unsigned ord = 0;
                            for (int k = 0; k < S.nrow[gs]; ++k) {
                                const int2 rw = S.u.rows[k][gs];
                                if (cand >= rw.y) ord += (unsigned)(rw.y - rw.x);
                                else { ord += (unsigned)(cand - rw.x); break; }
                            }
                            record_singular(P, make_err_key(ST_EDGE, ts + gs, ord), ou, ov, -1, -1, 2);
                        }
                        keep = o.size <= P.tol.lim_a;                                          // pipeline.py:358
                    }
                    const unsigned m = __ballot_sync(FULL, keep);
                    __syncwarp();                           // every lane has read its entry before the prefix is overwritten
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
            // ---- B: every lane walks its own candidate rows
            bool crowded = false;
            {
                int r = 0, pos = 0, end = 0;
#if EL_PREF_ROW
                if (nr > 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + S.u.rows[0][lane].x));
#endif
#if EL_WALK2
                // EL_WALK2 candidates of the row per iteration: a warp issues in order and every iteration ends in a
                // ballot, so with one record per iteration each of the ~33 candidates of a lane cost a full load latency.
                constexpr int K = EL_WALK2;
                for (;;) {
                    if (pos >= end && r < nr) {             // parked rows are non-empty: one step suffices
                        const int2 q = S.u.rows[r][lane];
                        pos = q.x; end = q.y; ++r;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + pos));
                    }
                    const int have = min(end - pos, K);     // candidates this lane takes in this iteration
                    if (!__any_sync(FULL, have > 0)) break;
                    if (pos + K < end) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + pos + K));
                    Atom av[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        av[k].x = av[k].y = av[k].z = 0.0; av[k].r2 = -1.0;
                        if (k < have) av[k] = load_atom(P.xyzr, pos + k);                       // (x, y, z, reach)
                    }
                    unsigned m[K];
                    unsigned any = 0;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const double dx = av[k].x - ux, dy = av[k].y - uy, dz = av[k].z - uz;
                        const double lims = av[k].r2 + ureach;
                        const bool pass = av[k].r2 >= 0.0 && (dx * dx + dy * dy) + dz * dz <= lims * lims;   // pipeline.py:341-344
                        m[k] = __ballot_sync(FULL, pass);
                        any |= m[k];
                    }
                    if (any) {
                        if (qn + 32 * K > EL_QCAP) {        // nearly full (dense cores): count exactly what this iteration queues,
                            int add = 0;                    // the queue is used to its last slot before a pass is given up
#pragma unroll
                            for (int k = 0; k < K; ++k) add += __popc(m[k]);
                            if (qn + add > EL_QCAP) {
                                settle();
                                if (qn + add > EL_QCAP) { crowded = true; break; }
                            }
                        }
#pragma unroll
                        for (int k = 0; k < K; ++k) {       // (a lane's candidates stay in ascending rank)
                            if ((m[k] >> lane) & 1u) {
                                const int at = qn + __popc(m[k] & lanemask_lt());
                                S.q_cand[at] = pos + k; S.q_gen[at] = (unsigned char)lane;
                            }
                            qn += __popc(m[k]);
                        }
                        __syncwarp();
                    }
                    pos += max(have, 0);
                }
#else
                for (;;) {
                    if (pos >= end && r < nr) {             // parked rows are non-empty: one step suffices
                        const int2 q = S.u.rows[r][lane];
                        pos = q.x; end = q.y; ++r;
#if EL_PREF_ROW
                        // the NEXT row's first line is requested while this row is walked (a row is ~2.5 records, i.e.
                        // one or two 128-byte lines, and the L1 is mostly shared memory here: most first touches miss)
                        if (r < nr) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + S.u.rows[r][lane].x));
#else
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + pos));
#endif
                    }
                    const bool have = pos < end;
                    if (!__any_sync(FULL, have)) break;
                    bool pass = false;
                    if (have) {
                        if (pos + EL_PREF_AHEAD < end) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.xyzr + pos + EL_PREF_AHEAD));
                        const Atom av = load_atom(P.xyzr, pos);                                 // (x, y, z, reach)
                        const double dx = av.x - ux, dy = av.y - uy, dz = av.z - uz;
                        const double lims = av.r2 + ureach;
                        pass = av.r2 >= 0.0 && (dx * dx + dy * dy) + dz * dz <= lims * lims;    // pipeline.py:341-344
                    }
                    const unsigned m = __ballot_sync(FULL, pass);
                    if (m) {
                        if (qn + 32 > EL_QCAP) {
                            settle();
                            if (qn + 32 > EL_QCAP) { crowded = true; break; }
                        }
                        if (pass) {
                            const int at = qn + __popc(m & lanemask_lt());
                            S.q_cand[at] = pos; S.q_gen[at] = (unsigned char)lane;
                        }
                        qn += __popc(m);
                        __syncwarp();
                    }
                    if (have) ++pos;
                }
#endif
            }
            if (crowded) {
                // more kept pairs than the queue holds: halve the pass and redo it; a single generator that still does
                // not fit is left to k_edges_heavy (count, allocate, write)
                __syncwarp();
                if (gb > 1) { gb = gb / 2; continue; }
                if (lane == 0) { P.deg[ts] = -1; atomicAdd(&P.ctr->n_heavy, 1u); }            // for k_edges_heavy
                ts += 1;
                gb = 32;
                continue;
            }
            settle();
            // ---- D: partner lists.  Count per generator, prefix, stable scatter (rounds in queue order, match_any
            // ranks the lanes of one generator inside a round), then one global atomicAdd and coalesced stores.
            if (qn > 0) {
                S.cnt[lane] = 0;
                __syncwarp();
                for (int x = lane; x < qn; x += 32) atomicAdd(&S.cnt[S.q_gen[x]], 1);
                __syncwarp();
                const int d = S.cnt[lane];
                const int incl = warp_incl_scan(d);
                S.off[lane + 1] = incl;
                if (lane == 0) S.off[0] = 0;
                if (d > MAXP) atomicOr(&P.ctr->overflow, 1u);                      // AXB_ERR_DENSITY
                if (d > 0) {
                    max_deg = max(max_deg, (unsigned)d);
                    pairs += (unsigned long long)d * (unsigned)(d - 1) / 2;
                }
                __syncwarp();
                S.cnt[lane] = incl - d;                                            // cursors
                __syncwarp();
                for (int x0 = 0; x0 < qn; x0 += 32) {
                    const int x = x0 + lane;
                    const bool valid = x < qn;
                    const int gs = valid ? (int)S.q_gen[x] : 32 + lane;            // idle lanes: unique keys
                    const unsigned peers = __match_any_sync(FULL, gs);
                    if (valid) {
                        S.u.sorted[S.cnt[gs] + __popc(peers & lanemask_lt())] = S.q_cand[x];
                    }
                    __syncwarp();
                    if (valid && (peers & lanemask_lt()) == 0u) S.cnt[gs] += __popc(peers);   // the group's first lane
                    __syncwarp();
                }
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(&P.ctr->n_pe, (unsigned)qn);
                base = __shfl_sync(FULL, base, 0);
                if ((unsigned long long)base + (unsigned)qn <= P.pe_cap) {
                    if (d > 0) {
                        P.adj_off[t] = base + (unsigned)(incl - d);
                        P.deg[t] = d;
                    }
                    for (int idx = lane; idx < qn; idx += 32) {
                        int gi = 0;                         // generator slot: last one with off <= idx
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1)
                            if (gi + step < 32 && S.off[gi + step] <= idx) gi += step;
                        P.pe_v[base + idx] = S.u.sorted[idx];
                        P.pe_u[base + idx] = ts + gi;
                    }
                } else if (lane == 0) {
                    atomicOr(&P.ctr->overflow, 1u << 4);   // potential-edge buffer too small: caller re-runs
                }
            }
            __syncwarp();
            ts += gb;
            gb = 32;
        }
    }
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

// The generators k_edges marked (deg == -1): a warp each, two sweeps (heavy_generator).
__global__ void __launch_bounds__(EL_WARPS * 32) k_edges_heavy(EstParams P, int rank_lo, int rank_hi) {
    extern __shared__ __align__(16) unsigned char s_raw_el[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    ELWarp &S = reinterpret_cast<ELWarp *>(s_raw_el)[warp];
    unsigned max_deg = 0;
    unsigned long long pairs = 0;
    for (int t = rank_lo + blockIdx.x * EL_WARPS + warp; t < rank_hi; t += gridDim.x * EL_WARPS) {
        if (P.deg[t] != -1) continue;
        double ux, uy, uz, ureach = -1.0;
        const int nr = lane_rows(P, S, t, lane, lane == 0, ux, uy, uz, ureach);
        S.nrow[lane] = nr;
        __syncwarp();
        const unsigned d = heavy_generator(P, S, t, lane);
        if (lane == 0) {
            if (d == 0) P.deg[t] = 0;
            if (d > (unsigned)MAXP) atomicOr(&P.ctr->overflow, 1u);                               // AXB_ERR_DENSITY
            max_deg = max(max_deg, d);
            pairs += (unsigned long long)d * (d - 1) / 2;
        }
        __syncwarp();
    }
    if (lane == 0 && max_deg) {
        atomicMax(&P.ctr->max_deg, max_deg);
        atomicAdd(&P.ctr->pair_bound, pairs);
    }
}

}  // namespace axb
