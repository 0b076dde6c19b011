/*
 * alpha_oracle.h -- CPU oracle for the alpha-complex hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * package's algorithm (alphax 0.1.0: pipeline.py, geometry.py, grid.py,
 * _arrays.py).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product
 * (paper_1908_05944_b200) never does.
 *
 * Parity status: PINNED.  The restatement is checked bit-for-bit against
 * outputs of the real Python reference generated in the build container
 * (tests/golden/ fixtures, made by tools/make_golden.py) and against the
 * reference's own known-answer fixtures (tests/test_oracle_golden.py).
 */
#ifndef ALPHA_ORACLE_H
#define ALPHA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirror the reference's exception types, errors.py:4-24) */
enum {
    AXO_OK = 0,
    AXO_EMPTY = 1,        /* EmptyInput            pipeline.py:226-227 */
    AXO_NONFINITE = 2,    /* NonFiniteCoordinate   pipeline.py:235-237 */
    AXO_DUPLICATE = 3,    /* DuplicateCenter       pipeline.py:238-244 */
    AXO_DEGENERATE = 4,   /* DegenerateSimplex     pipeline.py:263-266 */
    AXO_BAD_SIDE = 5,     /* ValueError            grid.py:113-117     */
    AXO_NOMEM = 6
};

/* what-selectors for the accessors below */
enum {
    AXO_K0 = 0, AXO_K1 = 1, AXO_K2 = 2, AXO_K3 = 3,   /* the complex      */
    AXO_PE = 4, AXO_PT = 5, AXO_PQ = 6                /* potential levels */
};

typedef struct axo_result axo_result;

/* geometry.py:161-181 + 122-158.  pts (m,k,3), r2 (m,k); k in 1..4.
 * Row 0 of each simplex must be the lowest-index ball (caller's job). */
void axo_ortho_batch(int64_t m, int k, const double *pts, const double *r2,
                     double eps_singular, double *centers, double *sizes,
                     uint8_t *singular);

/* grid.py:105-144.  Outputs: side, origin[3], dims[3], order[n], rank[n],
 * cells[n].  Returns AXO_OK / AXO_EMPTY / AXO_NONFINITE / AXO_BAD_SIDE. */
int axo_grid_build(int64_t n, const double *xyz, const double *radii,
                   double alpha, double *side, double *origin, int64_t *dims,
                   int64_t *order, int64_t *rank, int64_t *cells);

/* pipeline.py:286-313 restated for one query: AC2 of a simplex with given
 * ortho-centre/size against the 27-cell block.  Needs a grid handle, so it is
 * exposed through the full run below only. */

/* pipeline.py:571-628 (mode="grid").  chunk <= 0 means one chunk (chunk_size
 * None); threads is the worker count (OpenMP).  keep_potentials != 0 also
 * retains the whole-input potential levels (pipeline.py:640-709 views:
 * rows lexicographically sorted with cached centres/sizes).
 * Always returns a handle in *out (unless AXO_NOMEM); the status is also
 * stored in it. */
int axo_compute(int64_t n, const double *xyz, const double *radii,
                double alpha, double eps_abs, double eps_singular,
                int biomolecule, int64_t chunk, int threads,
                int keep_potentials, axo_result **out);

/* pipeline.py:530-555: ONE _chunk_pass over grid ranks [rank_lo, rank_hi) of the whole input (the
 * unit the reference hands to a worker; what one GPU slab computes).  Rows are sorted-unique. */
int axo_compute_range(int64_t n, const double *xyz, const double *radii,
                      double alpha, double eps_abs, double eps_singular,
                      int biomolecule, int64_t rank_lo, int64_t rank_hi, axo_result **out);

int axo_status(const axo_result *r);
/* for AXO_NONFINITE: verts[0] = ball; AXO_DUPLICATE: verts[0..1];
 * AXO_DEGENERATE: verts[0..nverts-1] (sorted ball indices). */
void axo_error(const axo_result *r, int64_t verts[4], int *nverts);
int64_t axo_count(const axo_result *r, int what);
const int64_t *axo_rows(const axo_result *r, int what);
const double *axo_centers(const axo_result *r, int what); /* AXO_PE..PQ */
const double *axo_sizes(const axo_result *r, int what);   /* AXO_PE..PQ */
/* per-stage seconds, summed over chunks, reference order
 * (grid, potential_edges, potential_triangles, potential_tets,
 *  prune_tets, prune_triangles, prune_edges, prune_vertices). */
void axo_stage_seconds(const axo_result *r, double out[8]);
void axo_free(axo_result *r);

#ifdef __cplusplus
}
#endif
#endif
