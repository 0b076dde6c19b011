// predicates.cuh -- fp64 geometric predicates with the reference's exact
// operation order (reference geometry.py:122-181, pipeline.py:286-313).
//
// Compile with -fmad=false: every multiply/add below is separately rounded.
// The ONLY fused operations are the explicit fma() calls of the Gram matrix,
// which reproduce what np.matmul (BLAS) computes at geometry.py:176:
//     G_ij = fma(D_i.z, D_j.z, fma(D_i.y, D_j.y, D_i.x * D_j.x)).
// Functions are __host__ __device__ so the same arithmetic can be unit-tested
// on the CPU against the golden vectors (tests/native/).
#pragma once

#include "common.cuh"

#include <math.h>

namespace axb {

#define AXB_HD __host__ __device__ __forceinline__

struct Ortho {
    double cx, cy, cz;   // ortho-centre
    double size;         // ortho-size
    bool singular;       // some |pivot| <= eps_singular
};

// squared distance with the reference's summation order ((dx^2 + dy^2) + dz^2)
AXB_HD double dist2(const Atom &a, const Atom &b) {
    double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return (dx * dx + dy * dy) + dz * dz;
}

// pipeline.py:343-344 / 400-401 / 460-461: reach pre-filter of a pair.
// reach < 0 encodes "not viable" (pipeline.py:323), which only matters for
// the edge stage; later stages only ever see viable balls.
AXB_HD bool reach_pair(const Atom &a, double reach_a, const Atom &b, double reach_b) {
    double lims = reach_a + reach_b;
    return dist2(a, b) <= lims * lims;
}

// k = 2 (geometry.py:161-181 with d = 1).  p0 must be the lower ball index.
AXB_HD Ortho ortho2(const Atom &p0, const Atom &p1, double eps_sing) {
    Ortho o;
    double Dx = p1.x - p0.x, Dy = p1.y - p0.y, Dz = p1.z - p0.z;
    double g = fma(Dz, Dz, fma(Dy, Dy, Dx * Dx));
    double a = 2.0 * g;
    double b = (((Dx * Dx + Dy * Dy) + Dz * Dz) + p0.r2) - p1.r2;
    o.singular = fabs(a) <= eps_sing;
    double lam = b / (o.singular ? 1.0 : a);
    o.cx = p0.x + lam * Dx;
    o.cy = p0.y + lam * Dy;
    o.cz = p0.z + lam * Dz;
    double ex = o.cx - p0.x, ey = o.cy - p0.y, ez = o.cz - p0.z;
    o.size = ((ex * ex + ey * ey) + ez * ez) - p0.r2;
    return o;
}

// Generic d x d partial-pivot solve (geometry.py:122-158), d = 2 or 3, fully
// unrolled so the matrix stays in registers (row swaps are predicated).
template <int d>
AXB_HD bool solve_pp(double (&A)[d][d], double (&b)[d], double (&x)[d], double eps_sing) {
    bool sing = false;
#pragma unroll
    for (int col = 0; col < d; ++col) {
        int piv = col;                       // first arg-max of |A[r][col]|, r >= col
        double best = fabs(A[col][col]);
#pragma unroll
        for (int r = col + 1; r < d; ++r) {
            double v = fabs(A[r][col]);
            if (v > best) { best = v; piv = r; }
        }
#pragma unroll
        for (int r = col + 1; r < d; ++r) {
            if (piv == r) {
#pragma unroll
                for (int c = 0; c < d; ++c) { double t = A[r][c]; A[r][c] = A[col][c]; A[col][c] = t; }
                double t = b[r]; b[r] = b[col]; b[col] = t;
            }
        }
        double pv = A[col][col];
        bool bad = fabs(pv) <= eps_sing;
        sing = sing || bad;
        double safe = bad ? 1.0 : pv;
#pragma unroll
        for (int r = col + 1; r < d; ++r) {
            double f = A[r][col] / safe;
#pragma unroll
            for (int c = col; c < d; ++c) A[r][c] = A[r][c] - f * A[col][c];
            b[r] = b[r] - f * b[col];
        }
    }
#pragma unroll
    for (int r = d - 1; r >= 0; --r) {
        double acc = b[r];
#pragma unroll
        for (int c = r + 1; c < d; ++c) acc = acc - A[r][c] * x[c];
        x[r] = acc / (sing ? 1.0 : A[r][r]);
    }
    return sing;
}

// k = 3 and k = 4.  p[0] must be the lowest ball index, the rest ascending.
template <int k>
AXB_HD Ortho orthoN(const Atom (&p)[k], double eps_sing) {
    constexpr int d = k - 1;
    double D[d][3], A[d][d], b[d], x[d];
#pragma unroll
    for (int i = 0; i < d; ++i) {
        D[i][0] = p[i + 1].x - p[0].x;
        D[i][1] = p[i + 1].y - p[0].y;
        D[i][2] = p[i + 1].z - p[0].z;
    }
#pragma unroll
    for (int i = 0; i < d; ++i)
#pragma unroll
        for (int j = i; j < d; ++j) {
            double g = fma(D[i][2], D[j][2], fma(D[i][1], D[j][1], D[i][0] * D[j][0]));
            A[i][j] = 2.0 * g;
            A[j][i] = A[i][j];               // products commute, so the mirror is bit-identical
        }
#pragma unroll
    for (int i = 0; i < d; ++i)
        b[i] = (((D[i][0] * D[i][0] + D[i][1] * D[i][1]) + D[i][2] * D[i][2]) + p[0].r2) - p[i + 1].r2;
    Ortho o;
    o.singular = solve_pp<d>(A, b, x, eps_sing);
    double sx = x[0] * D[0][0], sy = x[0] * D[0][1], sz = x[0] * D[0][2];
#pragma unroll
    for (int i = 1; i < d; ++i) {
        sx = sx + x[i] * D[i][0];
        sy = sy + x[i] * D[i][1];
        sz = sz + x[i] * D[i][2];
    }
    o.cx = p[0].x + sx;
    o.cy = p[0].y + sy;
    o.cz = p[0].z + sz;
    double ex = o.cx - p[0].x, ey = o.cy - p[0].y, ez = o.cz - p[0].z;
    o.size = ((ex * ex + ey * ey) + ez * ez) - p[0].r2;
    return o;
}

// conditional swap of (ball index, atom) pairs: sorting network building block
AXB_HD void cswap(int &ia, Atom &a, int &ib, Atom &b) {
    if (ia > ib) {
        int t = ia; ia = ib; ib = t;
        Atom s = a; a = b; b = s;
    }
}

AXB_HD Ortho ortho_edge(int i0, Atom a0, int i1, Atom a1, double eps_sing) {
    cswap(i0, a0, i1, a1);
    return ortho2(a0, a1, eps_sing);
}

AXB_HD Ortho ortho_tri(int i0, Atom a0, int i1, Atom a1, int i2, Atom a2, double eps_sing) {
    cswap(i0, a0, i1, a1);
    cswap(i1, a1, i2, a2);
    cswap(i0, a0, i1, a1);
    Atom p[3] = {a0, a1, a2};
    return orthoN<3>(p, eps_sing);
}

AXB_HD Ortho ortho_tet(int i0, Atom a0, int i1, Atom a1, int i2, Atom a2, int i3, Atom a3, double eps_sing) {
    cswap(i0, a0, i1, a1);
    cswap(i2, a2, i3, a3);
    cswap(i0, a0, i2, a2);
    cswap(i1, a1, i3, a3);
    cswap(i1, a1, i2, a2);
    Atom p[4] = {a0, a1, a2, a3};
    return orthoN<4>(p, eps_sing);
}

// grid.py:64-67 / 122-126: clamped cell coordinate of one axis
AXB_HD int cell_coord(double v, double origin, double side, int dim) {
    double q = floor((v - origin) / side);
    // clip in floating point first so absurd values cannot overflow the cast
    if (!(q > 0.0)) return 0;
    if (q >= (double)dim) return dim - 1;
    return (int)q;
}

// z layer inside the local table: global layer (clamped to the global grid exactly like the
// reference) minus the slab offset, clamped into the loaded range
AXB_HD int cell_coord_z(double v, const GridView &g) {
    int iz = cell_coord(v, g.oz, g.side, g.dz_glob) - g.z_lo;
    return iz < 0 ? 0 : (iz >= g.dz ? g.dz - 1 : iz);
}

#ifdef __CUDACC__
// Rank range [s, e) of the balls in cells x0..x1 of row (y, z): consecutive cells of a row are
// consecutive keys, and the balls are sorted by key, so it is one contiguous range.
// Dense mode reads the cell table; sparse mode binary-searches the sorted keys (the reference's
// searchsorted over occupied keys, grid.py:80-82).
__device__ __forceinline__ int rank_lower_bound(const GridView &g, long long key) {
    int lo = 0, hi = g.n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(g.skeys + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void row_range(const GridView &g, int x0, int x1, int y, int z, int &s, int &e) {
    if (g.cell_start) {
        const int row = g.dx * (y + g.dy * z);
        s = (int)__ldg(g.cell_start + row + x0);
        e = (int)__ldg(g.cell_start + row + x1 + 1);
    } else {
        const long long row = (long long)g.dx * ((long long)y + (long long)g.dy * (long long)z);
        s = rank_lower_bound(g, row + x0);
        e = rank_lower_bound(g, row + x1 + 1);
    }
}

// pipeline.py:286-313 for one simplex: true iff no non-incident ball of the 27-cell block around the
// ortho-centre has power distance < thr = size - eps_abs.  inc0..inc3 are the RANKS of the incident
// balls (-1 = unused).  Early exit at the first dominating ball.
//
// Exact trimming of the block: a ball p can only dominate if |p - c|^2 - r_p^2 < thr, hence only if
// |p - c|^2 < r2max + thr =: R2 (r2max = largest squared radius of the input).  Cells of the block
// whose nearest point is farther than sqrt(R2) from c (with a 1e-9 slack, far above any rounding)
// cannot hold such a ball and are skipped -- often most of the 27.  The boolean is unchanged.
__device__ __forceinline__ bool ac2_pass(const GridView &g, const Atom *__restrict__ atoms, double cx, double cy,
                                         double cz, double thr, double r2max, int inc0, int inc1, int inc2, int inc3) {
    double R2 = r2max + thr;
    if (!(R2 > 0.0)) return true;                       // dp >= -r_p^2 >= -r2max >= thr for every ball
    R2 = R2 * (1.0 + 1e-9) + 1e-9;
    const int ix = cell_coord(cx, g.ox, g.side, g.dx);
    const int iy = cell_coord(cy, g.oy, g.side, g.dy);
    const int iz = cell_coord_z(cz, g);
    // distances from c to the faces of its own cell (>= 0; c may sit outside a clamped border cell)
    const double xa = g.ox + (double)ix * g.side, ya = g.oy + (double)iy * g.side;
    const double za = g.oz + (double)(iz + g.z_lo) * g.side;
    const double dxl = fmax(cx - xa, 0.0), dxh = fmax(xa + g.side - cx, 0.0);
    const double dyl = fmax(cy - ya, 0.0), dyh = fmax(ya + g.side - cy, 0.0);
    const double dzl = fmax(cz - za, 0.0), dzh = fmax(za + g.side - cz, 0.0);
    const double ox2 = fmax(fmax(xa - cx, cx - (xa + g.side)), 0.0);     // distance to the own cell itself (0 inside)
    const double oy2 = fmax(fmax(ya - cy, cy - (ya + g.side)), 0.0);
    const double oz2 = fmax(fmax(za - cz, cz - (za + g.side)), 0.0);
    const int y0 = max(iy - 1, 0), y1 = min(iy + 1, g.dy - 1);
    const int z0 = max(iz - 1, 0), z1 = min(iz + 1, g.dz - 1);
    for (int z = z0; z <= z1; ++z) {
        const double gz = z < iz ? dzl : (z > iz ? dzh : oz2);
        const double rem_z = R2 - gz * gz;
        if (rem_z < 0.0) continue;
        for (int y = y0; y <= y1; ++y) {
            const double gy = y < iy ? dyl : (y > iy ? dyh : oy2);
            const double rem = rem_z - gy * gy;
            if (rem < 0.0) continue;
            int x0 = ix, x1 = ix;
            if (ix > 0 && dxl * dxl <= rem) x0 = ix - 1;
            if (ix < g.dx - 1 && dxh * dxh <= rem) x1 = ix + 1;
            if (ox2 * ox2 > rem) {                       // even the own column is out of reach (clamped centre)
                if (x0 == ix && x1 == ix) continue;
            }
            int s, e;
            row_range(g, x0, x1, y, z, s, e);
            for (int t = s; t < e; ++t) {
                const double2 *q = reinterpret_cast<const double2 *>(atoms + t);
                double2 xy = __ldg(q), zr = __ldg(q + 1);
                double ddx = xy.x - cx, ddy = xy.y - cy, ddz = zr.x - cz;
                double dp = ((ddx * ddx + ddy * ddy) + ddz * ddz) - zr.y;
                // incident balls are masked out (pipeline.py:306-307); they sit at dp == size > thr up to rounding, so
                // the mask is only consulted in the rare branch
                if (dp < thr && !(t == inc0 || t == inc1 || t == inc2 || t == inc3)) return false;
            }
        }
    }
    return true;
}

// one 256-bit load per atom record (sm_100: LDG.E.256), read-only path
__device__ __forceinline__ Atom load_atom(const Atom *__restrict__ atoms, int t) {
    Atom a;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(a.z), "=d"(a.r2) : "l"(atoms + t));
    return a;
}

// ac2_pass with memory-level parallelism (dense cell table only).  The plain version above is a chain
// of dependent round trips: row bounds -> balls of the row -> next row ...  Here (1) the bounds of all
// nine rows of the 3x3x3 block are fetched back to back (straight-line code, clamped indices, so the 18
// loads are in flight together) and parked in a per-thread column of shared memory, (2) the balls of
// all rows are walked as ONE flattened sequence with the next AC2_DEPTH + 1 balls prefetched into L1 ahead
// of the ball being tested.  Same boolean as ac2_pass (same cells, same arithmetic, pipeline.py:286-313).
#ifndef AC2_DEPTH
#define AC2_DEPTH 3
#endif
#ifndef AC2_PAIR
#define AC2_PAIR 1           // two balls of the flattened sequence per iteration (a thread issues in order)
#endif
__device__ __forceinline__ bool ac2_pass_mlp(const GridView &g, const Atom *__restrict__ atoms, double cx, double cy,
                                             double cz, double thr, double r2max, int inc0, int inc1, int inc2, int inc3,
                                             int2 *rows, int stride) {
    double R2 = r2max + thr;
    if (!(R2 > 0.0)) return true;
    R2 = R2 * (1.0 + 1e-9) + 1e-9;
    const int ix = cell_coord(cx, g.ox, g.side, g.dx);
    const int iy = cell_coord(cy, g.oy, g.side, g.dy);
    const int iz = cell_coord_z(cz, g);
    const double xa = g.ox + (double)ix * g.side, ya = g.oy + (double)iy * g.side;
    const double za = g.oz + (double)(iz + g.z_lo) * g.side;
    const double dxl = fmax(cx - xa, 0.0), dxh = fmax(xa + g.side - cx, 0.0);
    const double dyl = fmax(cy - ya, 0.0), dyh = fmax(ya + g.side - cy, 0.0);
    const double dzl = fmax(cz - za, 0.0), dzh = fmax(za + g.side - cz, 0.0);
    const double ox2 = fmax(fmax(xa - cx, cx - (xa + g.side)), 0.0);
    const double oy2 = fmax(fmax(ya - cy, cy - (ya + g.side)), 0.0);
    const double oz2 = fmax(fmax(za - cz, cz - (za + g.side)), 0.0);
    const double dxl2 = dxl * dxl, dxh2 = dxh * dxh, ox22 = ox2 * ox2;
    int sr[9], er[9];
#pragma unroll
    for (int oz = -1; oz <= 1; ++oz) {
        const int z = iz + oz;
        const double gz = oz < 0 ? dzl : (oz > 0 ? dzh : oz2);
        const double rem_z = R2 - gz * gz;
        const bool zok = z >= 0 && z < g.dz && rem_z >= 0.0;
#pragma unroll
        for (int oy = -1; oy <= 1; ++oy) {
            const int k = (oz + 1) * 3 + (oy + 1);
            const int y = iy + oy;
            const double gy = oy < 0 ? dyl : (oy > 0 ? dyh : oy2);
            const double rem = rem_z - gy * gy;
            bool ok = zok && y >= 0 && y < g.dy && rem >= 0.0;
            int x0 = ix, x1 = ix;
            if (ix > 0 && dxl2 <= rem) x0 = ix - 1;
            if (ix < g.dx - 1 && dxh2 <= rem) x1 = ix + 1;
            if (ox22 > rem && x0 == ix && x1 == ix) ok = false;
            const int row = ok ? g.dx * (y + g.dy * z) : 0;
            const int a = ok ? row + x0 : 0, b = ok ? row + x1 + 1 : 0;
            sr[k] = (int)__ldg(g.cell_start + a);
            er[k] = (int)__ldg(g.cell_start + b);
        }
    }
    // only the non-empty rows are parked (trimming and sparse regions leave several of the nine empty), so the
    // walk switches rows exactly once per row that holds balls
    // ... and in the order of their distance from the centre's own row: a dominating ball is most likely a close one, and
    // the walk ends at the first (at alpha = 1.4 two thirds of the potential tets and nearly all free triangles are dominated)
    int nr = 0;
#ifndef AC2_CENTER_FIRST
#define AC2_CENTER_FIRST 1
#endif
#if AC2_CENTER_FIRST
    constexpr int ORD[9] = {4, 3, 5, 1, 7, 0, 2, 6, 8};
#else
    constexpr int ORD[9] = {0, 1, 2, 3, 4, 5, 6, 7, 8};
#endif
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const int k = ORD[q];
        if (er[k] > sr[k]) {
            rows[nr * stride] = make_int2(sr[k], er[k]);
            ++nr;
        }
    }
    // flattened walk over the balls of all rows
    int r = -1, pos = 0, end = 0;
    auto next = [&]() -> int {
        if (pos >= end) {
            if (r + 1 >= nr) return -1;                   // exhausted (and stays so: r never leaves the parked rows)
            ++r;
            const int2 q = rows[r * stride];
            pos = q.x; end = q.y;
        }
        return pos++;
    };
#ifndef AC2_PREFETCH
#define AC2_PREFETCH 1
#endif
#if AC2_PREFETCH
    // The balls ahead are requested with prefetch.global.L1 (no destination register), the ball under test is
    // loaded when it is needed and hits L1: only two integers travel down the queue per step instead of whole
    // 32-byte records (the record queue spent a quarter of the kernel's instructions on register moves).
    auto prefetch = [&](int t) { asm volatile("prefetch.global.L1 [%0];" ::"l"(atoms + t)); };
    int tq[AC2_DEPTH + 1];
#pragma unroll
    for (int d = 0; d <= AC2_DEPTH; ++d) {
        tq[d] = next();
        if (tq[d] >= 0) prefetch(tq[d]);
    }
#if AC2_PAIR
    // two balls of the flattened sequence per iteration (AC2_DEPTH >= 3: two under test, two requested)
    static_assert(!AC2_PAIR || AC2_DEPTH >= 3, "AC2_PAIR needs a queue of four");
    while (tq[0] >= 0) {
        const int t0 = tq[0], t1 = tq[1];
        const Atom a = load_atom(atoms, t0);
        const Atom b = load_atom(atoms, t1 >= 0 ? t1 : t0);
#pragma unroll
        for (int d = 0; d + 2 <= AC2_DEPTH; ++d) tq[d] = tq[d + 2];
        tq[AC2_DEPTH - 1] = next();
        if (tq[AC2_DEPTH - 1] >= 0) prefetch(tq[AC2_DEPTH - 1]);
        tq[AC2_DEPTH] = next();
        if (tq[AC2_DEPTH] >= 0) prefetch(tq[AC2_DEPTH]);
        const double ax = a.x - cx, ay = a.y - cy, az = a.z - cz;
        const double bx = b.x - cx, by = b.y - cy, bz = b.z - cz;
        const double dpa = ((ax * ax + ay * ay) + az * az) - a.r2;
        const double dpb = ((bx * bx + by * by) + bz * bz) - b.r2;
        if (dpa < thr && !(t0 == inc0 || t0 == inc1 || t0 == inc2 || t0 == inc3)) return false;   // incident balls are masked (pipeline.py:306-307)
        if (t1 >= 0 && dpb < thr && !(t1 == inc0 || t1 == inc1 || t1 == inc2 || t1 == inc3)) return false;
    }
#else
    while (tq[0] >= 0) {
        const int t = tq[0];
        const Atom a = load_atom(atoms, t);
#pragma unroll
        for (int d = 0; d < AC2_DEPTH; ++d) tq[d] = tq[d + 1];
        tq[AC2_DEPTH] = next();
        if (tq[AC2_DEPTH] >= 0) prefetch(tq[AC2_DEPTH]);
        const double ddx = a.x - cx, ddy = a.y - cy, ddz = a.z - cz;
        const double dp = ((ddx * ddx + ddy * ddy) + ddz * ddz) - a.r2;
        if (dp < thr && !(t == inc0 || t == inc1 || t == inc2 || t == inc3)) return false;   // incident balls are masked (pipeline.py:306-307)
    }
#endif
#else
    int tq[AC2_DEPTH];
    Atom aq[AC2_DEPTH];
#pragma unroll
    for (int d = 0; d < AC2_DEPTH; ++d) {
        tq[d] = next();
        if (tq[d] >= 0) aq[d] = load_atom(atoms, tq[d]);
    }
    while (tq[0] >= 0) {
        const int t = tq[0];
        const Atom a = aq[0];
#pragma unroll
        for (int d = 0; d + 1 < AC2_DEPTH; ++d) { tq[d] = tq[d + 1]; aq[d] = aq[d + 1]; }
        tq[AC2_DEPTH - 1] = next();
        if (tq[AC2_DEPTH - 1] >= 0) aq[AC2_DEPTH - 1] = load_atom(atoms, tq[AC2_DEPTH - 1]);
        const double ddx = a.x - cx, ddy = a.y - cy, ddz = a.z - cz;
        const double dp = ((ddx * ddx + ddy * ddy) + ddz * ddz) - a.r2;
        if (dp < thr && !(t == inc0 || t == inc1 || t == inc2 || t == inc3)) return false;   // incident balls are masked (pipeline.py:306-307)
    }
#endif
    return true;
}
#endif

}  // namespace axb
