/*
 * alpha_oracle.c -- CPU oracle (TEST INFRASTRUCTURE, never shipped on the
 * product path; see alpha_oracle.h).
 *
 * Plain-C restatement of the reference package alphax 0.1.0.  Citations are
 * into /root/reference/pkg/src/alphax/ (pipe = pipeline.py, geom =
 * geometry.py, grid = grid.py, arr = _arrays.py).  The arithmetic follows the
 * reference operation by operation so that the simplex sets AND the cached
 * ortho-centres/sizes are bit-identical; the only fused operation is the Gram
 * matrix (np.matmul -> BLAS, an FMA chain x*x, then y, then z), everything
 * else is separately rounded.  Build with -ffp-contract=off.
 *
 * Parity: pinned against the Python reference by tests/golden (see header).
 */
#define _GNU_SOURCE
#include "alpha_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ utils */

typedef struct { int64_t *v; int64_t n, cap; } ivec;
typedef struct { double *v; int64_t n, cap; } dvec;

static void iv_reserve(ivec *a, int64_t extra) {
    if (a->n + extra > a->cap) {
        int64_t c = a->cap ? a->cap * 2 : 64;
        while (c < a->n + extra) c *= 2;
        a->v = (int64_t *)realloc(a->v, (size_t)c * sizeof(int64_t));
        a->cap = c;
    }
}
static void iv_push(ivec *a, int64_t x) { iv_reserve(a, 1); a->v[a->n++] = x; }
static void iv_free(ivec *a) { free(a->v); a->v = NULL; a->n = a->cap = 0; }
static void dv_reserve(dvec *a, int64_t extra) {
    if (a->n + extra > a->cap) {
        int64_t c = a->cap ? a->cap * 2 : 64;
        while (c < a->n + extra) c *= 2;
        a->v = (double *)realloc(a->v, (size_t)c * sizeof(double));
        a->cap = c;
    }
}
static void dv_push(dvec *a, double x) { dv_reserve(a, 1); a->v[a->n++] = x; }
static void dv_free(dvec *a) { free(a->v); a->v = NULL; a->n = a->cap = 0; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* row comparators: lexicographic on k int64 columns (arr:12-16, np.unique
 * axis=0 ordering) */
static int cmp_rows(const void *a, const void *b, void *kp) {
    int k = *(const int *)kp;
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    for (int c = 0; c < k; ++c) {
        if (x[c] < y[c]) return -1;
        if (x[c] > y[c]) return 1;
    }
    return 0;
}

/* arr:12-16 unique_rows: sort rows in place, drop duplicates, return count */
static int64_t sort_unique_rows(int64_t *rows, int64_t m, int k) {
    if (m == 0) return 0;
    qsort_r(rows, (size_t)m, (size_t)k * sizeof(int64_t), cmp_rows, &k);
    int64_t w = 1;
    for (int64_t i = 1; i < m; ++i) {
        if (cmp_rows(rows + (size_t)i * k, rows + (size_t)(w - 1) * k, &k) != 0) {
            if (w != i) memcpy(rows + (size_t)w * k, rows + (size_t)i * k, (size_t)k * sizeof(int64_t));
            ++w;
        }
    }
    return w;
}

/* arr:24-30 rows_in against a sorted duplicate-free table */
static int row_in_sorted(const int64_t *row, const int64_t *table, int64_t m, int k) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        int c = cmp_rows(table + (size_t)mid * k, row, &k);
        if (c == 0) return 1;
        if (c < 0) lo = mid + 1; else hi = mid;
    }
    return 0;
}

static void sort_small(int64_t *v, int k) { /* np.sort(axis=1) on a row */
    for (int i = 1; i < k; ++i) {
        int64_t x = v[i];
        int j = i - 1;
        while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; }
        v[j + 1] = x;
    }
}

/* --------------------------------------------------------------- geometry */

/* geom:122-158 + geom:161-181 for ONE simplex of k balls (k = 2..4).
 * p[i] = centre of the i-th ball in ascending ball index, q[i] = r_i^2. */
static void ortho_one(int k, const double p[4][3], const double q[4],
                      double eps_singular, double centre[3], double *size,
                      int *singular) {
    int d = k - 1;
    double D[3][3], A[3][3], b[3], x[3];
    int sing = 0;
    if (k == 1) { /* geom:173-174 */
        centre[0] = p[0][0]; centre[1] = p[0][1]; centre[2] = p[0][2];
        *size = -q[0];
        *singular = 0;
        return;
    }
    for (int i = 0; i < d; ++i)           /* geom:175 diffs */
        for (int c = 0; c < 3; ++c) D[i][c] = p[i + 1][c] - p[0][c];
    for (int i = 0; i < d; ++i)           /* geom:176 a = 2 * (diffs @ diffs^T) */
        for (int j = 0; j < d; ++j) {
            double g = D[i][0] * D[j][0];
            g = fma(D[i][1], D[j][1], g);
            g = fma(D[i][2], D[j][2], g);
            A[i][j] = 2.0 * g;
        }
    for (int i = 0; i < d; ++i) {         /* geom:177 rhs */
        double s = D[i][0] * D[i][0] + D[i][1] * D[i][1];
        s = s + D[i][2] * D[i][2];
        b[i] = (s + q[0]) - q[i + 1];
    }
    for (int col = 0; col < d; ++col) {   /* geom:135-151 elimination */
        int piv = col;
        double best = fabs(A[col][col]);
        for (int r = col + 1; r < d; ++r) {   /* argmax: first maximum wins */
            double v = fabs(A[r][col]);
            if (v > best) { best = v; piv = r; }
        }
        if (piv != col) {
            for (int c = 0; c < d; ++c) { double t = A[piv][c]; A[piv][c] = A[col][c]; A[col][c] = t; }
            double t = b[piv]; b[piv] = b[col]; b[col] = t;
        }
        double pv = A[col][col];
        int bad = fabs(pv) <= eps_singular;    /* geom:145 */
        if (bad) sing = 1;
        double safe = bad ? 1.0 : pv;          /* geom:147 */
        for (int r = col + 1; r < d; ++r) {
            double f = A[r][col] / safe;
            for (int c = col; c < d; ++c) A[r][c] = A[r][c] - f * A[col][c];
            b[r] = b[r] - f * b[col];
        }
    }
    for (int r = d - 1; r >= 0; --r) {    /* geom:152-157 back substitution */
        double acc = b[r];
        for (int c = r + 1; c < d; ++c) acc = acc - A[r][c] * x[c];
        x[r] = acc / (sing ? 1.0 : A[r][r]);
    }
    for (int c = 0; c < 3; ++c) {         /* geom:179 */
        double s = x[0] * D[0][c];
        for (int i = 1; i < d; ++i) s = s + x[i] * D[i][c];
        centre[c] = p[0][c] + s;
    }
    {                                      /* geom:180 */
        double e0 = centre[0] - p[0][0], e1 = centre[1] - p[0][1], e2 = centre[2] - p[0][2];
        double s = e0 * e0 + e1 * e1;
        s = s + e2 * e2;
        *size = s - q[0];
    }
    *singular = sing;
}

void axo_ortho_batch(int64_t m, int k, const double *pts, const double *r2,
                     double eps_singular, double *centers, double *sizes,
                     uint8_t *singular) {
    for (int64_t s = 0; s < m; ++s) {
        double p[4][3], q[4];
        int sg;
        for (int i = 0; i < k; ++i) {
            for (int c = 0; c < 3; ++c) p[i][c] = pts[((size_t)s * k + i) * 3 + c];
            q[i] = r2[(size_t)s * k + i];
        }
        ortho_one(k, p, q, eps_singular, centers + (size_t)s * 3, sizes + s, &sg);
        singular[s] = (uint8_t)sg;
    }
}

/* ------------------------------------------------------------------- grid */

typedef struct {
    int64_t n;
    double side, origin[3];
    int64_t dims[3];
    int64_t *order, *rank, *cells;     /* grid:35-37 */
    int64_t nocc, *occ, *off;          /* grid:38-39 */
} grid_t;

typedef struct { int64_t key, idx; } keyidx;
static int cmp_keyidx(const void *a, const void *b) {
    const keyidx *x = (const keyidx *)a, *y = (const keyidx *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);  /* stable == tie-break by index */
}

static int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

static void grid_free(grid_t *g) {
    free(g->order); free(g->rank); free(g->cells); free(g->occ); free(g->off);
    memset(g, 0, sizeof(*g));
}

/* grid:105-144 */
static int grid_build(grid_t *g, int64_t n, const double *xyz, const double *radii, double alpha, int64_t *bad) {
    memset(g, 0, sizeof(*g));
    if (n == 0) return AXO_EMPTY;
    for (int64_t i = 0; i < n; ++i)
        if (!(isfinite(xyz[3 * i]) && isfinite(xyz[3 * i + 1]) && isfinite(xyz[3 * i + 2]))) {
            if (bad) *bad = i;
            return AXO_NONFINITE;
        }
    double rmax = radii[0];
    for (int64_t i = 1; i < n; ++i) if (radii[i] > rmax) rmax = radii[i];
    double side_sq = rmax * rmax + alpha;
    if (side_sq <= 0.0) return AXO_BAD_SIDE;
    double side = sqrt(side_sq);
    double lo[3], hi[3];
    for (int c = 0; c < 3; ++c) lo[c] = hi[c] = xyz[c];
    for (int64_t i = 1; i < n; ++i)
        for (int c = 0; c < 3; ++c) {
            double v = xyz[3 * i + c];
            if (v < lo[c]) lo[c] = v;
            if (v > hi[c]) hi[c] = v;
        }
    g->n = n; g->side = side;
    for (int c = 0; c < 3; ++c) {
        g->origin[c] = lo[c];
        g->dims[c] = (int64_t)floor((hi[c] - lo[c]) / side) + 1;
    }
    g->order = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    g->rank = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    g->cells = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    keyidx *ki = (keyidx *)malloc((size_t)n * sizeof(keyidx));
    for (int64_t i = 0; i < n; ++i) {
        int64_t c3[3];
        for (int c = 0; c < 3; ++c)
            c3[c] = clampi((int64_t)floor((xyz[3 * i + c] - lo[c]) / side), 0, g->dims[c] - 1);
        int64_t lin = c3[0] + g->dims[0] * (c3[1] + g->dims[1] * c3[2]);
        g->cells[i] = lin;
        ki[i].key = lin; ki[i].idx = i;
    }
    qsort(ki, (size_t)n, sizeof(keyidx), cmp_keyidx);
    int64_t nocc = 0;
    for (int64_t t = 0; t < n; ++t) {
        g->order[t] = ki[t].idx;
        g->rank[ki[t].idx] = t;
        if (t == 0 || ki[t].key != ki[t - 1].key) ++nocc;
    }
    g->nocc = nocc;
    g->occ = (int64_t *)malloc((size_t)nocc * sizeof(int64_t));
    g->off = (int64_t *)malloc((size_t)(nocc + 1) * sizeof(int64_t));
    int64_t w = 0;
    for (int64_t t = 0; t < n; ++t)
        if (t == 0 || ki[t].key != ki[t - 1].key) { g->occ[w] = ki[t].key; g->off[w] = t; ++w; }
    g->off[nocc] = n;
    free(ki);
    return AXO_OK;
}

int axo_grid_build(int64_t n, const double *xyz, const double *radii,
                   double alpha, double *side, double *origin, int64_t *dims,
                   int64_t *order, int64_t *rank, int64_t *cells) {
    grid_t g;
    int st = grid_build(&g, n, xyz, radii, alpha, NULL);
    if (st != AXO_OK) { grid_free(&g); return st; }
    *side = g.side;
    for (int c = 0; c < 3; ++c) { origin[c] = g.origin[c]; dims[c] = g.dims[c]; }
    memcpy(order, g.order, (size_t)n * sizeof(int64_t));
    memcpy(rank, g.rank, (size_t)n * sizeof(int64_t));
    memcpy(cells, g.cells, (size_t)n * sizeof(int64_t));
    grid_free(&g);
    return AXO_OK;
}

/* grid:69-88 neighbor_indices: ranks (positions in `order`) of the balls in
 * the (2r+1)^3 block around cell (cx,cy,cz), ascending.  Cells along x are
 * consecutive keys, so each (y,z) row is one run over the occupied-key table. */
static void block_ranks(const grid_t *g, int64_t cx, int64_t cy, int64_t cz, int r, ivec *out) {
    out->n = 0;
    int64_t x0 = cx - r < 0 ? 0 : cx - r, x1 = cx + r > g->dims[0] - 1 ? g->dims[0] - 1 : cx + r;
    int64_t y0 = cy - r < 0 ? 0 : cy - r, y1 = cy + r > g->dims[1] - 1 ? g->dims[1] - 1 : cy + r;
    int64_t z0 = cz - r < 0 ? 0 : cz - r, z1 = cz + r > g->dims[2] - 1 ? g->dims[2] - 1 : cz + r;
    for (int64_t z = z0; z <= z1; ++z)
        for (int64_t y = y0; y <= y1; ++y) {
            int64_t klo = x0 + g->dims[0] * (y + g->dims[1] * z);
            int64_t khi = x1 + g->dims[0] * (y + g->dims[1] * z);
            int64_t a = 0, b = g->nocc;           /* first occupied key >= klo */
            while (a < b) { int64_t m = a + (b - a) / 2; if (g->occ[m] < klo) a = m + 1; else b = m; }
            for (; a < g->nocc && g->occ[a] <= khi; ++a)
                for (int64_t t = g->off[a]; t < g->off[a + 1]; ++t) iv_push(out, t);
        }
}

static void delinearize(const grid_t *g, int64_t lin, int64_t c3[3]) { /* grid:48-51 */
    c3[0] = lin % g->dims[0];
    int64_t rest = lin / g->dims[0];
    c3[1] = rest % g->dims[1];
    c3[2] = rest / g->dims[1];
}

/* --------------------------------------------------------------- pipeline */

typedef struct {
    int64_t n;
    const double *xyz;        /* (n,3) */
    double *r2;               /* pipe:590 */
    double *reach;            /* pipe:324 */
    uint8_t *viable;          /* pipe:323 */
    grid_t grid;
    double alpha, eps_abs, eps_sing, lim_a; /* lim_a = alpha + eps_abs */
    int biomolecule;
} ctx_t;

typedef struct {
    int status;
    int64_t verts[4];
    int nverts;
} err_t;

/* one level of potential simplices as produced by a chunk (pipe:316-479) */
typedef struct {
    ivec rows;    /* m*k sorted ball indices */
    dvec cents;   /* m*3 */
    dvec sizes;   /* m   */
} level_t;

static void level_free(level_t *l) { iv_free(&l->rows); dv_free(&l->cents); dv_free(&l->sizes); }

static void gather(const ctx_t *c, const int64_t *row, int k, double p[4][3], double q[4]) {
    for (int i = 0; i < k; ++i) {
        for (int a = 0; a < 3; ++a) p[i][a] = c->xyz[3 * row[i] + a];
        q[i] = c->r2[row[i]];
    }
}

static double dist2(const ctx_t *c, int64_t a, int64_t b) { /* (c[a]-c[b])^2 summed left to right */
    double dx = c->xyz[3 * a] - c->xyz[3 * b];
    double dy = c->xyz[3 * a + 1] - c->xyz[3 * b + 1];
    double dz = c->xyz[3 * a + 2] - c->xyz[3 * b + 2];
    double s = dx * dx + dy * dy;
    return s + dz * dz;
}

static int reach_ok(const ctx_t *c, int64_t a, int64_t b) { /* pipe:343-344, 400-401, 460-461 */
    double lims = c->reach[a] + c->reach[b];
    return dist2(c, a, b) <= lims * lims;
}

static void set_degenerate(err_t *e, const int64_t *row, int k) {
    if (e->status != AXO_OK) return;
    e->status = AXO_DEGENERATE;
    e->nverts = k;
    for (int i = 0; i < k; ++i) e->verts[i] = row[i];
}

/* pipe:286-313 for one simplex */
static int ac2_one(const ctx_t *c, const int64_t *row, int k, const double pt[3], double size, ivec *scratch) {
    const grid_t *g = &c->grid;
    int64_t c3[3];
    for (int a = 0; a < 3; ++a)   /* grid:64-67 */
        c3[a] = clampi((int64_t)floor((pt[a] - g->origin[a]) / g->side), 0, g->dims[a] - 1);
    block_ranks(g, c3[0], c3[1], c3[2], 1, scratch);
    if (scratch->n == 0) return 1;          /* pipe:302-303 */
    double best = INFINITY;
    for (int64_t i = 0; i < scratch->n; ++i) {
        int64_t nb = g->order[scratch->v[i]];
        int inc = 0;
        for (int j = 0; j < k; ++j) if (row[j] == nb) inc = 1;
        if (inc) continue;                   /* pipe:310-311 */
        double dx = c->xyz[3 * nb] - pt[0], dy = c->xyz[3 * nb + 1] - pt[1], dz = c->xyz[3 * nb + 2] - pt[2];
        double s = dx * dx + dy * dy;
        s = s + dz * dz;
        double dp = s - c->r2[nb];           /* pipe:309 */
        if (dp < best) best = dp;
    }
    return best >= size - c->eps_abs;        /* pipe:312 */
}

typedef struct {
    ivec k[4];              /* kept simplices of the chunk, flattened rows */
    level_t pot[3];         /* potential edges / triangles / tets */
    double t[8];
    err_t err;
    int err_stage;          /* ordering key for the first failure */
} chunk_out;

static void chunk_free(chunk_out *o) {
    for (int d = 0; d < 4; ++d) iv_free(&o->k[d]);
    for (int d = 0; d < 3; ++d) level_free(&o->pot[d]);
}

/* pipe:530-555 _chunk_pass */
static void chunk_pass(const ctx_t *c, int64_t lo, int64_t hi, chunk_out *o) {
    const grid_t *g = &c->grid;
    const int64_t *order = g->order, *rank = g->rank;
    ivec nb = {0}, gen = {0}, par = {0};
    ivec scratch = {0};
    double t0;
    memset(o, 0, sizeof(*o));

    /* ---- pipe:316-359 potential edges */
    t0 = now_s();
    {
        ivec cu = {0}, cv = {0};
        for (int64_t t = lo; t < hi; ++t) {
            int64_t u = order[t];
            if (!c->viable[u]) continue;
            int64_t c3[3];
            delinearize(g, g->cells[u], c3);
            block_ranks(g, c3[0], c3[1], c3[2], 2, &nb);
            for (int64_t i = 0; i < nb.n; ++i) {
                if (nb.v[i] <= t) continue;         /* pipe:338 rank > t */
                int64_t v = order[nb.v[i]];
                if (reach_ok(c, v, u) && c->viable[v]) { iv_push(&cu, u); iv_push(&cv, v); }
            }
        }
        int64_t m = cu.n;
        double *cen = (double *)malloc((size_t)(m ? m : 1) * 3 * sizeof(double));
        double *siz = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
        for (int64_t i = 0; i < m; ++i) {           /* pipe:355-356 */
            int64_t row[2] = {cu.v[i], cv.v[i]};
            double p[4][3], q[4]; int sg;
            sort_small(row, 2);
            gather(c, row, 2, p, q);
            ortho_one(2, p, q, c->eps_sing, cen + 3 * i, siz + i, &sg);
            if (sg) set_degenerate(&o->err, row, 2);   /* first in list order, pipe:357 */
        }
        if (o->err.status == AXO_OK)
            for (int64_t i = 0; i < m; ++i)
                if (siz[i] <= c->lim_a) {           /* pipe:358 */
                    int64_t row[2] = {cu.v[i], cv.v[i]};
                    sort_small(row, 2);
                    iv_push(&o->pot[0].rows, row[0]); iv_push(&o->pot[0].rows, row[1]);
                    for (int a = 0; a < 3; ++a) dv_push(&o->pot[0].cents, cen[3 * i + a]);
                    dv_push(&o->pot[0].sizes, siz[i]);
                    iv_push(&gen, cu.v[i]); iv_push(&par, cv.v[i]);
                }
        free(cen); free(siz); iv_free(&cu); iv_free(&cv);
    }
    o->t[1] += now_s() - t0;
    if (o->err.status != AXO_OK) goto done;

    /* ---- pipe:373-423 potential triangles.  gen/par are already ordered by
     * (rank[gen], rank[par]) (pipe:362-370) because generators were visited
     * in rank order and each block lists its balls in ascending rank. */
    ivec tu = {0}, tv = {0}, tw = {0}, thi = {0};
    t0 = now_s();
    {
        ivec cu = {0}, cv = {0}, cw = {0};
        for (int64_t s = 0; s < gen.n;) {
            int64_t e = s;
            while (e < gen.n && gen.v[e] == gen.v[s]) ++e;
            for (int64_t i = s; i < e; ++i)               /* np.triu_indices(k, 1) order */
                for (int64_t j = i + 1; j < e; ++j)
                    if (reach_ok(c, par.v[i], par.v[j])) {
                        iv_push(&cu, gen.v[s]); iv_push(&cv, par.v[i]); iv_push(&cw, par.v[j]);
                    }
            s = e;
        }
        int64_t m = cu.n;
        uint8_t *ok = (uint8_t *)calloc((size_t)(m ? m : 1), 1);
        for (int64_t i = 0; i < m; ++i) {               /* pipe:412-415 */
            int64_t row[2] = {cv.v[i], cw.v[i]};
            double p[4][3], q[4], cen[3], siz; int sg;
            sort_small(row, 2);
            gather(c, row, 2, p, q);
            ortho_one(2, p, q, c->eps_sing, cen, &siz, &sg);
            if (sg) set_degenerate(&o->err, row, 2);
            ok[i] = siz <= c->lim_a;
        }
        if (o->err.status == AXO_OK) {
            double *cen = (double *)malloc((size_t)(m ? m : 1) * 3 * sizeof(double));
            double *siz = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
            for (int64_t i = 0; i < m; ++i) {           /* pipe:417-419 */
                if (!ok[i]) continue;
                int64_t row[3] = {cu.v[i], cv.v[i], cw.v[i]};
                double p[4][3], q[4]; int sg;
                sort_small(row, 3);
                gather(c, row, 3, p, q);
                ortho_one(3, p, q, c->eps_sing, cen + 3 * i, siz + i, &sg);
                if (sg) set_degenerate(&o->err, row, 3);
            }
            if (o->err.status == AXO_OK)
                for (int64_t i = 0; i < m; ++i)
                    if (ok[i] && siz[i] <= c->lim_a) {  /* pipe:420-423 */
                        int64_t row[3] = {cu.v[i], cv.v[i], cw.v[i]};
                        sort_small(row, 3);
                        for (int a = 0; a < 3; ++a) iv_push(&o->pot[1].rows, row[a]);
                        for (int a = 0; a < 3; ++a) dv_push(&o->pot[1].cents, cen[3 * i + a]);
                        dv_push(&o->pot[1].sizes, siz[i]);
                        iv_push(&tu, cu.v[i]); iv_push(&tv, cv.v[i]); iv_push(&tw, cw.v[i]);
                        int64_t rv = rank[cv.v[i]], rw = rank[cw.v[i]];
                        iv_push(&thi, rv > rw ? rv : rw);
                    }
            free(cen); free(siz);
        }
        free(ok); iv_free(&cu); iv_free(&cv); iv_free(&cw);
    }
    o->t[2] += now_s() - t0;
    if (o->err.status != AXO_OK) { iv_free(&tu); iv_free(&tv); iv_free(&tw); iv_free(&thi); goto done; }

    /* ---- pipe:426-479 potential tets */
    t0 = now_s();
    if (tu.n && gen.n) {
        ivec ct = {0}, cx = {0};
        /* triangles are already grouped by generator in rank order
         * (pipe:437-440: stable argsort of rank[tri_u] over a list built in
         * that order); adjacency group of the same generator (pipe:435-436) */
        int64_t es = 0;
        for (int64_t s = 0; s < tu.n;) {
            int64_t e = s;
            while (e < tu.n && tu.v[e] == tu.v[s]) ++e;
            while (es < gen.n && gen.v[es] != tu.v[s]) ++es;
            int64_t ee = es;
            while (ee < gen.n && gen.v[ee] == tu.v[s]) ++ee;
            for (int64_t t = s; t < e; ++t)            /* pipe:447-451, row-major nonzero */
                for (int64_t xi = es; xi < ee; ++xi)
                    if (rank[par.v[xi]] > thi.v[t]) { iv_push(&ct, t); iv_push(&cx, par.v[xi]); }
            s = e;
        }
        int64_t m = ct.n;
        uint8_t *ok = (uint8_t *)calloc((size_t)(m ? m : 1), 1);
        for (int64_t i = 0; i < m; ++i) {              /* pipe:458-463 */
            int64_t t = ct.v[i], x = cx.v[i];
            ok[i] = reach_ok(c, x, tv.v[t]) && reach_ok(c, x, tw.v[t]);
        }
        for (int pass = 0; pass < 2 && o->err.status == AXO_OK; ++pass) {   /* pipe:467-474 */
            for (int64_t i = 0; i < m; ++i) {
                if (!ok[i]) continue;
                int64_t t = ct.v[i];
                int64_t row[2] = {pass == 0 ? tv.v[t] : tw.v[t], cx.v[i]};
                double p[4][3], q[4], cen[3], siz; int sg;
                sort_small(row, 2);
                gather(c, row, 2, p, q);
                ortho_one(2, p, q, c->eps_sing, cen, &siz, &sg);
                if (sg) set_degenerate(&o->err, row, 2);
                ok[i] = siz <= c->lim_a;
            }
        }
        if (o->err.status == AXO_OK) {
            double *cen = (double *)malloc((size_t)(m ? m : 1) * 3 * sizeof(double));
            double *siz = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
            for (int64_t i = 0; i < m; ++i) {          /* pipe:475-477 */
                if (!ok[i]) continue;
                int64_t t = ct.v[i];
                int64_t row[4] = {tu.v[t], tv.v[t], tw.v[t], cx.v[i]};
                double p[4][3], q[4]; int sg;
                sort_small(row, 4);
                gather(c, row, 4, p, q);
                ortho_one(4, p, q, c->eps_sing, cen + 3 * i, siz + i, &sg);
                if (sg) set_degenerate(&o->err, row, 4);
            }
            if (o->err.status == AXO_OK)
                for (int64_t i = 0; i < m; ++i)
                    if (ok[i] && siz[i] <= c->lim_a) { /* pipe:478-479 */
                        int64_t t = ct.v[i];
                        int64_t row[4] = {tu.v[t], tv.v[t], tw.v[t], cx.v[i]};
                        sort_small(row, 4);
                        for (int a = 0; a < 4; ++a) iv_push(&o->pot[2].rows, row[a]);
                        for (int a = 0; a < 3; ++a) dv_push(&o->pot[2].cents, cen[3 * i + a]);
                        dv_push(&o->pot[2].sizes, siz[i]);
                    }
            free(cen); free(siz);
        }
        free(ok); iv_free(&ct); iv_free(&cx);
    }
    o->t[3] += now_s() - t0;
    iv_free(&tu); iv_free(&tv); iv_free(&tw); iv_free(&thi);
    if (o->err.status != AXO_OK) goto done;

    /* ---- pipe:482-527 top-down pruning */
    {
        /* step 2: tets (pipe:496-497) */
        t0 = now_s();
        int64_t mq = o->pot[2].sizes.n;
        for (int64_t i = 0; i < mq; ++i)
            if (ac2_one(c, o->pot[2].rows.v + 4 * i, 4, o->pot[2].cents.v + 3 * i, o->pot[2].sizes.v[i], &scratch))
                for (int a = 0; a < 4; ++a) iv_push(&o->k[3], o->pot[2].rows.v[4 * i + a]);
        o->t[4] += now_s() - t0;

        /* steps 3 and 4: triangles, then edges (pipe:501-513) */
        for (int dim = 2; dim >= 1; --dim) {
            t0 = now_s();
            int k = dim + 1, ku = dim + 2;
            const ivec *up = &o->k[dim + 1];
            int64_t mu = up->n / ku;
            ivec faces = {0};                         /* arr:33-40 faces_of */
            for (int drop = 0; drop < ku; ++drop)
                for (int64_t i = 0; i < mu; ++i)
                    for (int a = 0; a < ku; ++a)
                        if (a != drop) iv_push(&faces, up->v[ku * i + a]);
            int64_t nf = sort_unique_rows(faces.v, faces.n / k, k);
            faces.n = nf * k;
            level_t *lv = &o->pot[dim - 1];
            int64_t m = lv->sizes.n;
            for (int64_t i = 0; i < m; ++i) {
                const int64_t *row = lv->rows.v + (size_t)k * i;
                if (row_in_sorted(row, faces.v, nf, k)) continue;      /* not free */
                if (ac2_one(c, row, k, lv->cents.v + 3 * i, lv->sizes.v[i], &scratch))
                    for (int a = 0; a < k; ++a) iv_push(&faces, row[a]);
            }
            int64_t nk = sort_unique_rows(faces.v, faces.n / k, k);
            faces.n = nk * k;
            o->k[dim] = faces;
            o->t[4 + (3 - dim)] += now_s() - t0;
        }

        /* step 5: vertices (pipe:516-526) */
        t0 = now_s();
        if (c->biomolecule) {
            for (int64_t t = lo; t < hi; ++t) iv_push(&o->k[0], order[t]);
        } else {
            ivec ends = {0};
            for (int64_t i = 0; i < o->k[1].n; ++i) iv_push(&ends, o->k[1].v[i]);
            int64_t ne = sort_unique_rows(ends.v, ends.n, 1);
            ends.n = ne;
            for (int64_t t = lo; t < hi; ++t) {
                int64_t v = order[t];
                if (!(-c->r2[v] <= c->lim_a)) continue;            /* pipe:520 */
                if (row_in_sorted(&v, ends.v, ne, 1)) continue;    /* pipe:522 */
                if (ac2_one(c, &v, 1, c->xyz + 3 * v, -c->r2[v], &scratch)) iv_push(&ends, v);
            }
            o->k[0] = ends;
        }
        int64_t n0 = sort_unique_rows(o->k[0].v, o->k[0].n, 1);
        o->k[0].n = n0;
        o->t[7] += now_s() - t0;
    }
done:
    iv_free(&nb); iv_free(&gen); iv_free(&par); iv_free(&scratch);
}

/* ----------------------------------------------------------------- result */

struct axo_result {
    int status;
    int64_t verts[4];
    int nverts;
    int64_t cnt[7];
    int64_t *rows[7];
    double *cents[7];
    double *sizes[7];
    double t[8];
};

int axo_status(const axo_result *r) { return r->status; }
void axo_error(const axo_result *r, int64_t verts[4], int *nverts) {
    for (int i = 0; i < 4; ++i) verts[i] = r->verts[i];
    *nverts = r->nverts;
}
int64_t axo_count(const axo_result *r, int what) { return r->cnt[what]; }
const int64_t *axo_rows(const axo_result *r, int what) { return r->rows[what]; }
const double *axo_centers(const axo_result *r, int what) { return r->cents[what]; }
const double *axo_sizes(const axo_result *r, int what) { return r->sizes[what]; }
void axo_stage_seconds(const axo_result *r, double out[8]) { memcpy(out, r->t, sizeof(r->t)); }
void axo_free(axo_result *r) {
    if (!r) return;
    for (int i = 0; i < 7; ++i) { free(r->rows[i]); free(r->cents[i]); free(r->sizes[i]); }
    free(r);
}

/* pipe:224-245 validate_input on arrays: finite check, then exact duplicate
 * centres via np.lexsort((z, y, x)) + adjacent compare. */
typedef struct { double x, y, z; int64_t i; } cidx;
static int cmp_cidx(const void *a, const void *b) {
    const cidx *p = (const cidx *)a, *q = (const cidx *)b;
    if (p->x != q->x) return p->x < q->x ? -1 : 1;
    if (p->y != q->y) return p->y < q->y ? -1 : 1;
    if (p->z != q->z) return p->z < q->z ? -1 : 1;
    return p->i < q->i ? -1 : (p->i > q->i ? 1 : 0);
}
static int validate(int64_t n, const double *xyz, const double *radii, axo_result *r) {
    if (n <= 0) return AXO_EMPTY;
    for (int64_t i = 0; i < n; ++i)
        if (!(isfinite(xyz[3 * i]) && isfinite(xyz[3 * i + 1]) && isfinite(xyz[3 * i + 2]) && isfinite(radii[i]))) {
            r->verts[0] = i; r->nverts = 1;
            return AXO_NONFINITE;
        }
    cidx *s = (cidx *)malloc((size_t)n * sizeof(cidx));
    for (int64_t i = 0; i < n; ++i) { s[i].x = xyz[3 * i]; s[i].y = xyz[3 * i + 1]; s[i].z = xyz[3 * i + 2]; s[i].i = i; }
    qsort(s, (size_t)n, sizeof(cidx), cmp_cidx);
    int st = AXO_OK;
    for (int64_t t = 1; t < n; ++t)
        if (s[t].x == s[t - 1].x && s[t].y == s[t - 1].y && s[t].z == s[t - 1].z) {
            int64_t i = s[t - 1].i, j = s[t].i;
            r->verts[0] = i < j ? i : j; r->verts[1] = i < j ? j : i; r->nverts = 2;
            st = AXO_DUPLICATE;
            break;
        }
    free(s);
    return st;
}

/* sort a potential level lexicographically, carrying centres/sizes
 * (pipe:635-637 _sorted_level) */
typedef struct { const int64_t *rows; int k; } permctx;
static int cmp_perm(const void *a, const void *b, void *cp) {
    const permctx *pc = (const permctx *)cp;
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    return cmp_rows(pc->rows + (size_t)i * pc->k, pc->rows + (size_t)j * pc->k, (void *)&pc->k);
}

static int compute_impl(int64_t n, const double *xyz, const double *radii,
                double alpha, double eps_abs, double eps_singular,
                int biomolecule, int64_t chunk, int threads,
                int keep_potentials, int64_t range_lo, int64_t range_hi, axo_result **out) {
    axo_result *r = (axo_result *)calloc(1, sizeof(axo_result));
    if (!r) return AXO_NOMEM;
    *out = r;
    r->status = validate(n, xyz, radii, r);
    if (r->status != AXO_OK) return r->status;

    ctx_t c;
    memset(&c, 0, sizeof(c));
    c.n = n; c.xyz = xyz; c.alpha = alpha; c.eps_abs = eps_abs; c.eps_sing = eps_singular;
    c.lim_a = alpha + eps_abs;
    c.biomolecule = biomolecule;
    double t0 = now_s();
    int64_t bad = -1;
    r->status = grid_build(&c.grid, n, xyz, radii, alpha, &bad);
    r->t[0] = now_s() - t0;
    if (r->status != AXO_OK) { grid_free(&c.grid); return r->status; }
    c.r2 = (double *)malloc((size_t)n * sizeof(double));
    c.reach = (double *)malloc((size_t)n * sizeof(double));
    c.viable = (uint8_t *)malloc((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        c.r2[i] = radii[i] * radii[i];                 /* pipe:590 */
        double lim = c.r2[i] + alpha + eps_abs;        /* pipe:322 */
        c.viable[i] = lim >= 0.0;                      /* pipe:323 */
        c.reach[i] = sqrt(lim > 0.0 ? lim : 0.0);      /* pipe:324 */
    }

    if (chunk <= 0 || chunk > n) chunk = n;            /* pipe:598 */
    int64_t nchunks = (n + chunk - 1) / chunk;
    if (range_lo >= 0) nchunks = 1;                    /* one explicit _chunk_pass(lo, hi), pipe:530 */
    chunk_out *parts = (chunk_out *)calloc((size_t)nchunks, sizeof(chunk_out));
    if (threads < 1) threads = 1;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
    for (int64_t ci = 0; ci < nchunks; ++ci) {
        int64_t lo = ci * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (range_lo >= 0) { lo = range_lo; hi = range_hi < n ? range_hi : n; }
        chunk_pass(&c, lo, hi, &parts[ci]);
    }

    /* first failing chunk in submission order (pool.map yields in order, pipe:609) */
    for (int64_t ci = 0; ci < nchunks && r->status == AXO_OK; ++ci)
        if (parts[ci].err.status != AXO_OK) {
            r->status = parts[ci].err.status;
            r->nverts = parts[ci].err.nverts;
            memcpy(r->verts, parts[ci].err.verts, sizeof(r->verts));
        }

    if (r->status == AXO_OK) {
        for (int d = 0; d < 4; ++d) {                  /* pipe:611-614 */
            int k = d + 1;
            int64_t tot = 0;
            for (int64_t ci = 0; ci < nchunks; ++ci) tot += parts[ci].k[d].n;
            int64_t *all = (int64_t *)malloc((size_t)(tot ? tot : 1) * sizeof(int64_t));
            int64_t w = 0;
            for (int64_t ci = 0; ci < nchunks; ++ci) {
                memcpy(all + w, parts[ci].k[d].v, (size_t)parts[ci].k[d].n * sizeof(int64_t));
                w += parts[ci].k[d].n;
            }
            r->cnt[d] = sort_unique_rows(all, tot / k, k);
            r->rows[d] = all;
        }
        if (keep_potentials)
            for (int d = 0; d < 3; ++d) {
                int k = d + 2;
                int64_t m = 0;
                for (int64_t ci = 0; ci < nchunks; ++ci) m += parts[ci].pot[d].sizes.n;
                int64_t *rows = (int64_t *)malloc((size_t)(m ? m : 1) * k * sizeof(int64_t));
                double *cen = (double *)malloc((size_t)(m ? m : 1) * 3 * sizeof(double));
                double *siz = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
                int64_t w = 0;
                for (int64_t ci = 0; ci < nchunks; ++ci) {
                    level_t *lv = &parts[ci].pot[d];
                    memcpy(rows + (size_t)w * k, lv->rows.v, (size_t)lv->rows.n * sizeof(int64_t));
                    memcpy(cen + (size_t)w * 3, lv->cents.v, (size_t)lv->cents.n * sizeof(double));
                    memcpy(siz + w, lv->sizes.v, (size_t)lv->sizes.n * sizeof(double));
                    w += lv->sizes.n;
                }
                int64_t *perm = (int64_t *)malloc((size_t)(m ? m : 1) * sizeof(int64_t));
                for (int64_t i = 0; i < m; ++i) perm[i] = i;
                permctx pc = {rows, k};
                qsort_r(perm, (size_t)m, sizeof(int64_t), cmp_perm, &pc);
                int64_t *rows2 = (int64_t *)malloc((size_t)(m ? m : 1) * k * sizeof(int64_t));
                double *cen2 = (double *)malloc((size_t)(m ? m : 1) * 3 * sizeof(double));
                double *siz2 = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
                for (int64_t i = 0; i < m; ++i) {
                    memcpy(rows2 + (size_t)i * k, rows + (size_t)perm[i] * k, (size_t)k * sizeof(int64_t));
                    memcpy(cen2 + (size_t)i * 3, cen + (size_t)perm[i] * 3, 3 * sizeof(double));
                    siz2[i] = siz[perm[i]];
                }
                free(rows); free(cen); free(siz); free(perm);
                r->cnt[4 + d] = m; r->rows[4 + d] = rows2; r->cents[4 + d] = cen2; r->sizes[4 + d] = siz2;
            }
    }
    for (int64_t ci = 0; ci < nchunks; ++ci) {
        for (int s = 0; s < 8; ++s) r->t[s] += parts[ci].t[s];
        chunk_free(&parts[ci]);
    }
    free(parts);
    free(c.r2); free(c.reach); free(c.viable);
    grid_free(&c.grid);
    return r->status;
}

int axo_compute(int64_t n, const double *xyz, const double *radii,
                double alpha, double eps_abs, double eps_singular,
                int biomolecule, int64_t chunk, int threads,
                int keep_potentials, axo_result **out) {
    return compute_impl(n, xyz, radii, alpha, eps_abs, eps_singular, biomolecule, chunk, threads,
                        keep_potentials, -1, -1, out);
}

int axo_compute_range(int64_t n, const double *xyz, const double *radii,
                      double alpha, double eps_abs, double eps_singular,
                      int biomolecule, int64_t rank_lo, int64_t rank_hi, axo_result **out) {
    if (rank_lo < 0) rank_lo = 0;
    return compute_impl(n, xyz, radii, alpha, eps_abs, eps_singular, biomolecule, 0, 1, 0, rank_lo, rank_hi, out);
}
