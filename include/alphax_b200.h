/*
 * alphax_b200.h -- C ABI of the B200-native alpha-complex hot path.
 *
 * The reference package (alphax 0.1.0) has no FFI layer: its boundary for this
 * path is the Python function compute_alpha_complex (reference
 * pkg/src/alphax/pipeline.py:571-628) plus the standalone stage operations
 * (pipeline.py:640-731, grid.py:105-144).  This header is the C-ABI a binding
 * for that boundary would call; each entry point names the reference code it
 * replaces.  Plain pointers and sizes only; no exceptions cross the ABI; every
 * function returns an axb_status.  All device work is hand-written CUDA for
 * sm_100a (paper_1908_05944_b200/csrc), launched on the context's stream.
 *
 * Memory: the caller owns all device memory.  Scratch comes from one caller-
 * provided arena (axb_ctx_set_arena); when it is too small a call returns
 * AXB_ERR_ARENA and axb_arena_needed() says how much would have been enough so
 * far -- grow and call again.  Inputs/outputs are caller buffers.
 */
#ifndef ALPHAX_B200_H
#define ALPHAX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum axb_status {
    AXB_OK = 0,
    AXB_ERR_BAD_ARG = 1,
    AXB_ERR_CUDA = 2,          /* a CUDA runtime call failed; see axb_last_message */
    AXB_ERR_ARENA = 3,         /* scratch arena too small; see axb_arena_needed    */
    AXB_ERR_EMPTY = 4,         /* EmptyInput            (pipeline.py:226-227)      */
    AXB_ERR_NONFINITE = 5,     /* NonFiniteCoordinate   (pipeline.py:235-237)      */
    AXB_ERR_DUPLICATE = 6,     /* DuplicateCenter       (pipeline.py:238-244)      */
    AXB_ERR_DEGENERATE = 7,    /* DegenerateSimplex     (pipeline.py:263-266)      */
    AXB_ERR_BAD_SIDE = 8,      /* ValueError, non-positive squared cell side (grid.py:113-117) */
    AXB_ERR_GRID_TOO_LARGE = 9,/* dense cell table would exceed the supported size */
    AXB_ERR_DENSITY = 10,      /* a ball has more than AXB_MAX_PARTNERS potential-edge partners */
    AXB_ERR_STATE = 11,        /* stages called out of order                       */
    AXB_ERR_INTERNAL = 12
} axb_status;

#define AXB_MAX_PARTNERS 1023

typedef struct axb_ctx axb_ctx;

/* run parameters: PipelineConfig + TolerancePolicy (pipeline.py:55-83, geometry.py:22-37) */
typedef struct axb_params {
    double alpha;          /* A^2, compared as size <= alpha + eps_abs */
    double eps_abs;        /* TolerancePolicy.eps_abs      */
    double eps_singular;   /* TolerancePolicy.eps_singular */
    int32_t biomolecule;   /* PipelineConfig.biomolecule_mode */
    int32_t reserved;
} axb_params;

/* grid geometry (grid.py:30-39) */
typedef struct axb_grid_info {
    double origin[3];
    double cell_side;
    int64_t dims[3];
    int64_t n_cells;
    int64_t n_balls;
} axb_grid_info;

/* one z-slab of a global grid (multi-GPU sharding): geometry of the GLOBAL grid
 * (grid.py:112-121 evaluated on the whole input) and the loaded cell layers [z_lo, z_hi) */
typedef struct axb_slab {
    double origin[3];
    double cell_side;
    int64_t dims[3];
    int64_t z_lo, z_hi;
} axb_slab;

/* what-selectors */
enum { AXB_K0 = 0, AXB_K1 = 1, AXB_K2 = 2, AXB_K3 = 3, AXB_PE = 4, AXB_PT = 5, AXB_PQ = 6 };

/* stage indices of axb_stage_ms: the reference's STAGE_NAMES (pipeline.py:43-52)
 * with "io" replaced by prune_vertices (cli.py:210 folds it into prune_edges),
 * plus this implementation's canonicalisation (count/scan/scatter) and export
 * (in-bucket sort + int64 rows) stages. */
enum {
    AXB_ST_GRID = 0, AXB_ST_POT_EDGES, AXB_ST_POT_TRIANGLES, AXB_ST_POT_TETS,
    AXB_ST_PRUNE_TETS, AXB_ST_PRUNE_TRIANGLES, AXB_ST_PRUNE_EDGES, AXB_ST_PRUNE_VERTICES,
    AXB_ST_CANONICAL, AXB_ST_EXPORT, AXB_ST_COUNT
};

/* ---- context ---------------------------------------------------------- */
int axb_version(void);
const char *axb_status_name(int status);
int axb_ctx_create(axb_ctx **out, int device);
void axb_ctx_destroy(axb_ctx *ctx);
int axb_ctx_set_stream(axb_ctx *ctx, void *cuda_stream);      /* cudaStream_t; NULL = default */
int axb_ctx_set_arena(axb_ctx *ctx, void *dev_ptr, size_t bytes);
size_t axb_arena_needed(const axb_ctx *ctx);
size_t axb_arena_used(const axb_ctx *ctx);
/* a conservative first guess for the arena size (bytes) */
size_t axb_arena_hint(int64_t n, double alpha, double r_max);
const char *axb_last_message(const axb_ctx *ctx);
/* AXB_ERR_NONFINITE: verts[0]; AXB_ERR_DUPLICATE: verts[0..1];
 * AXB_ERR_DEGENERATE: verts[0..nverts-1] ascending ball indices. */
int axb_last_error(const axb_ctx *ctx, int *status, int64_t verts[4], int *nverts);
/* What ranks of a sharded run need to agree on ONE error (the one the reference would raise for the whole
 * input, pipeline.py:238-244 / 357, 414, 419, 477).  AXB_ERR_DEGENERATE: *key = (stage << 60 | generator rank in
 * this context's grid order << 29 | ordinal); the smallest key over all ranks -- after adding the slab's first
 * global grid rank << 29 -- is the solve the reference meets first.  AXB_ERR_DUPLICATE: xyz = the shared centre
 * (the reference reports the smallest one in (x, y, z) order).  Ball indices from axb_last_error are GLOBAL
 * (mapped through d_global_index) when the context holds a slab. */
int axb_last_error_detail(const axb_ctx *ctx, uint64_t *key, double xyz[3]);

/* ---- the hot path, stage by stage ------------------------------------- */
/* validate_input + build_grid_arrays (pipeline.py:224-245, grid.py:105-144).
 * d_xyz: n x 3 row-major f64, d_radii: n f64, both DEVICE pointers. */
int axb_grid_build(axb_ctx *ctx, int64_t n, const double *d_xyz, const double *d_radii,
                   const axb_params *params);
/* Same for ONE SLAB of a larger input: the caller fixes the global grid geometry and passes only
 * the balls whose cell layer lies in [z_lo, z_hi), in ascending global ball index;
 * d_global_index (n int64, may be NULL) renames them in the exported rows.  This is the paper's
 * partition strategy (PAPER 4.6) / the reference's chunk ownership (pipeline.py:10-15) across GPUs. */
int axb_grid_build_slab(axb_ctx *ctx, int64_t n, const double *d_xyz, const double *d_radii,
                        const int64_t *d_global_index, const axb_params *params, const axb_slab *slab);
/* grid ranks [rank_lo, rank_hi) of the balls in cell layers [z_own_lo, z_own_hi) -- the generator
 * range to pass to axb_potential for the layers this slab OWNS (the rest is halo) */
int axb_slab_rank_range(axb_ctx *ctx, int64_t z_own_lo, int64_t z_own_hi, int64_t *rank_lo, int64_t *rank_hi);
int axb_grid_get_info(const axb_ctx *ctx, axb_grid_info *out);
/* order / rank / ball_cells of the reference Grid as int64 DEVICE arrays (any may be NULL) */
int axb_grid_export(axb_ctx *ctx, int64_t *d_order, int64_t *d_rank, int64_t *d_ball_cells);

/* _chunk_potential_edges / _triangles / _tets (pipeline.py:316-479) for the
 * generators at grid ranks [rank_lo, rank_hi); (0, n) is the whole input. */
int axb_potential(axb_ctx *ctx, int64_t rank_lo, int64_t rank_hi);
/* counts[0..2] = potential edges, triangles, tets */
int axb_potential_counts(const axb_ctx *ctx, int64_t counts[3]);
/* one potential level as the reference's PotentialLevel (pipeline.py:86-106):
 * rows (m, dim+1) int64 ascending ball indices, lexicographically sorted,
 * with cached centres (m,3) / sizes (m,) (either may be NULL).  DEVICE buffers. */
int axb_potential_export(axb_ctx *ctx, int what, int64_t *d_rows, double *d_centers, double *d_sizes);

/* ---- the standalone stage operations (pipeline.py:640-731) on resident or caller-supplied levels ---------- */
/* potential_edges (pipeline.py:640-646): stage one alone; the edge level stays resident */
int axb_potential_edges(axb_ctx *ctx, int64_t rank_lo, int64_t rank_hi);
/* potential triangles + tets (_chunk_potential_triangles / _tets, pipeline.py:373-479) from the RESIDENT edge level,
 * whichever way it got there (axb_potential_edges or axb_potential_import_edges) */
int axb_potential_simplices(axb_ctx *ctx);
/* potential_triangles(edges, ...) / prune(potentials, ...) consume the ROWS the caller passes (pipeline.py:658-667,
 * 712-731): replace the resident edge level by d_rows (m, 2) int64 ball indices, any row order (needs the grid);
 * replace the resident triangle and tet lists by rows (m_t, 3) / (m_q, 4) (needs the edge level; every edge of every
 * row must be in it).  DEVICE buffers.  AXB_ERR_BAD_ARG for rows that are not simplices of the input. */
int axb_potential_import_edges(axb_ctx *ctx, const int64_t *d_rows, int64_t m);
int axb_potential_import_simplices(axb_ctx *ctx, const int64_t *d_tri_rows, int64_t m_t, const int64_t *d_tet_rows, int64_t m_q);
/* potential_tets(triangles, ...) as the reference's standalone form (pipeline.py:670-709): every given triangle
 * (d_tri_rows: (m_t, 3) ascending ball indices, rows in lexicographic order) is extended by the larger ball indices
 * of the 5x5x5 cell block around its first ball whose three new faces are all in the list; kept when the
 * ortho-size is at most alpha + slack.  The given triangles and the resulting tets become the resident lists. */
int axb_potential_tets_from_triangles(axb_ctx *ctx, const int64_t *d_tri_rows, int64_t m_t);
/* _ac2_mask (pipeline.py:286-313) of one resident potential level (what = AXB_PE / AXB_PT / AXB_PQ), in the row
 * order of axb_potential_export: d_mask[e] = 1 iff no non-incident ball of the 27 cells around the ortho-centre
 * has power distance < size - eps_abs.  DEVICE buffer of uint8. */
int axb_ac2_mask(axb_ctx *ctx, int what, uint8_t *d_mask);

/* ---- alpha sweep with re-use ----------------------------------------------
 * Ortho-sizes and AC2 outcomes do not depend on alpha, and the potential levels at alpha are subsets of those at
 * a larger alpha.  axb_sweep_prepare: after axb_grid_build + axb_potential(0, n) at the LARGEST alpha of a sweep,
 * evaluate size and AC2 once for every listed simplex.  axb_sweep_prune(alpha), alpha <= that largest value: the
 * pruning stage for `alpha` from those arrays (the reference's own comparisons re-evaluated with alpha's reach and
 * limit, pipeline.py:322-324, 341-344, 358, 415, 420, 478), followed by axb_canonicalize / axb_export as usual;
 * may be called for any number of alphas.  Results are bit-identical to independent runs at each alpha. */
int axb_sweep_prepare(axb_ctx *ctx);
int axb_sweep_prune(axb_ctx *ctx, double alpha);
/* The sweep as a filtration, when its alphas are known up front (ascending, k <= 254, all <= the alpha of the
 * preparation): axb_sweep_rank gives every listed simplex the index of the first alpha at which the reference keeps it
 * -- own(s) = first index at which s is potential (if AC2(s)), a(s) = min(own(s), a(listed cofaces)), top-down, once --
 * and axb_sweep_select(index) marks { s : a(s) <= index }: one threshold pass per alpha, then axb_canonicalize /
 * axb_export.  AXB_ERR_STATE from axb_sweep_rank: a face of a listed tet is not a listed triangle (possible only by
 * rounding); use axb_sweep_prune. */
int axb_sweep_rank(axb_ctx *ctx, const double *alphas, int k);
int axb_sweep_select(axb_ctx *ctx, int index);

/* _prune_levels (pipeline.py:482-527): AC2 at every ortho-centre, inheritance of faces */
int axb_prune(axb_ctx *ctx);
/* canonical sort + dedup (pipeline.py:611-614, _arrays.py:12-16); counts[d] = simplices of dimension d */
int axb_canonicalize(axb_ctx *ctx, int64_t counts[4]);
/* the four canonical int64 arrays of AlphaComplex (pipeline.py:117-130) into DEVICE buffers
 * sized from axb_canonicalize's counts: (k0,), (k1,2), (k2,3), (k3,4) */
int axb_export(axb_ctx *ctx, int64_t *d_vertices, int64_t *d_edges, int64_t *d_triangles, int64_t *d_tets);

/* waits for the stream and reports deferred device-side flags (singular solves, internal checks);
 * call it after axb_export before trusting DEVICE output buffers (axb_export_host does it itself) */
int axb_sync_check(axb_ctx *ctx);

/* ---- the hot path in one call ------------------------------------------ */
/* compute_alpha_complex (pipeline.py:571-628, mode="grid") on DEVICE inputs:
 * grid_build -> potential(0,n) -> prune -> canonicalize. */
int axb_compute(axb_ctx *ctx, int64_t n, const double *d_xyz, const double *d_radii,
                const axb_params *params, int64_t counts[4]);
/* axb_compute + axb_export in one call when the caller can bound the list lengths (e.g. from the previous call on a
 * similar input: frames of a trajectory, repeated benchmark steps): the four int64 lists go straight into DEVICE buffers
 * of capacity[d] rows, and nothing waits for the host between the pruning stage and the last row -- one stream sync at the
 * very end instead of two plus the caller's allocation in between.  counts[d] = rows written.  AXB_ERR_STATE: a list was
 * longer than its buffer (counts[] holds the lengths; nothing in the buffers is valid): call axb_compute + axb_export. */
int axb_compute_into(axb_ctx *ctx, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *params,
                     int64_t *d_vertices, int64_t *d_edges, int64_t *d_triangles, int64_t *d_tets,
                     const int64_t capacity[4], int64_t counts[4]);
/* The same in two calls, so that the caller can allocate the buffers WHILE the GPU works: `start` returns after the edge
 * stage's sync with the triangle / tet and pruning kernels (two thirds of the step) still queued; `finish_into` queues
 * the canonical lists into the buffers and ends with the one sync that reads the row counts. */
int axb_compute_start(axb_ctx *ctx, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *params);
int axb_compute_finish_into(axb_ctx *ctx, int64_t *d_vertices, int64_t *d_edges, int64_t *d_triangles, int64_t *d_tets,
                            const int64_t capacity[4], int64_t counts[4]);
/* One z-slab of a sharded run in one call (what one GPU of a multi-GPU job executes):
 * axb_grid_build_slab -> potential simplices of the lower halo and of the OWNED layers [z_own_lo, z_own_hi) ->
 * prune -> canonicalize.  The slab emits exactly the kept simplices whose minimum-rank vertex (their generator,
 * pipeline.py:10-15) lies in an owned layer: it decides them completely on its own -- faces inherited from kept
 * simplices generated in the lower halo (pipeline.py:501-513) included, which is why the loaded layers must reach 2
 * below and 2 above the owned ones -- so the slabs' row lists are DISJOINT and their plain sorted merge is the
 * complex.  Rows exported afterwards carry global ball indices. */
int axb_compute_slab(axb_ctx *ctx, int64_t n, const double *d_xyz, const double *d_radii,
                     const int64_t *d_global_index, const axb_params *params, const axb_slab *slab,
                     int64_t z_own_lo, int64_t z_own_hi, int64_t counts[4]);
/* Same from HOST buffers: copies inputs to the arena, runs axb_compute. */
int axb_compute_host(axb_ctx *ctx, int64_t n, const double *h_xyz, const double *h_radii,
                     const axb_params *params, int64_t counts[4]);
/* Pipelined variant of axb_compute_host + axb_export_host: `begin` runs up to the potential stage and
 * returns row CAPACITIES for the four host arrays (tight upper bounds known at that point); the
 * caller allocates them (pinned memory makes the copies asynchronous) and calls `finish`, which
 * canonicalises every dimension as soon as it is final and copies it to the host on a second stream
 * while the remaining kernels run.  counts[d] <= capacity[d] rows of each array are valid.
 * The host arrays may be pageable: the DMA target is a pinned staging area owned by the context.
 * AXB_ERR_STATE from `finish` means a capacity bound did not hold (then use the two-call path). */
int axb_compute_host_begin(axb_ctx *ctx, int64_t n, const double *h_xyz, const double *h_radii,
                           const axb_params *params, int64_t capacity[4]);
int axb_compute_host_finish(axb_ctx *ctx, int64_t *h_vertices, int64_t *h_edges, int64_t *h_triangles,
                            int64_t *h_tets, int64_t counts[4]);
/* bytes the last axb_compute_host_finish moved device -> host: the rows cross PCIe as three bytes per
 * value while ball indices fit 24 bits (AXB_WIRE24=0 switches that off), else as int32 (ball indices
 * < 2^31), and host threads expand them to the int64 rows of the reference while later chunks are
 * still in flight (AXB_WIDEN_THREADS overrides the thread count) */
int64_t axb_last_d2h_bytes(const axb_ctx *ctx);
/* axb_export into HOST buffers (pinned or pageable). */
int axb_export_host(axb_ctx *ctx, int64_t *h_vertices, int64_t *h_edges, int64_t *h_triangles, int64_t *h_tets);

/* ---- merge of per-slab results ------------------------------------------- */
/* Sorted, duplicate-free union of m canonical rows of width k (1..4) with indices in [0, n_index):
 * the final np.unique of the reference (pipeline.py:611-614) for lists gathered from several slabs.
 * d_rows (m, k) and d_out (capacity m rows) are DEVICE int64; *count_out = rows written.
 * Reuses the scratch arena from the start (drops the state of a previous run). */
int axb_merge_rows(axb_ctx *ctx, int k, int64_t n_index, const int64_t *d_rows, int64_t m, int64_t *d_out,
                   int64_t *count_out);
/* The same for rows whose first index lies in [index_lo, index_hi): what one rank of a sharded run interleaves after
 * the rows were redistributed by index range (bucket arrays sized for the range, not for the whole job). */
int axb_merge_rows_range(axb_ctx *ctx, int k, int64_t index_lo, int64_t index_hi, const int64_t *d_rows, int64_t m,
                         int64_t *d_out, int64_t *count_out);

/* ---- canonical text document (a "next" row of SURVEY 8(f)) ---------------- */
/* The body of write_complex (reference io.py:228-236): one line "dim v0 [v1 [v2 [v3]]]\n" per
 * simplex in (dimension, lexicographic) order, from the four HOST int64 arrays.  Host threads, no
 * GPU.  *needed receives the byte count; with out == NULL only the size is computed; returns
 * AXB_ERR_ARENA if capacity is too small. */
int axb_format_complex(const int64_t counts[4], const int64_t *vertices, const int64_t *edges,
                       const int64_t *triangles, const int64_t *tets, char *out, int64_t capacity, int64_t *needed);

/* ---- measurement -------------------------------------------------------- */
/* Stage timing is recorded on request only, like the reference's optional `stage_times` dict
 * (pipeline.py:571, 595): on != 0 brackets every stage of the following runs with CUDA events (about 30
 * event records, 0.04-0.06 ms per run); off (the default) records nothing and axb_stage_ms reports zeros. */
int axb_set_stage_timing(axb_ctx *ctx, int on);
/* CUDA-event milliseconds per stage of the last run (zeros unless axb_set_stage_timing(ctx, 1)) */
int axb_stage_ms(const axb_ctx *ctx, float out[AXB_ST_COUNT]);
/* number of kernels this library launched since the context was created */
int64_t axb_kernel_launches(const axb_ctx *ctx);

/* ---- predicate probes (unit tests of the device arithmetic) ------------- */
/* geometry.py:161-181 on the device: pts (m,k,3), r2 (m,k), DEVICE pointers */
int axb_ortho_batch(axb_ctx *ctx, int64_t m, int k, const double *d_pts, const double *d_r2,
                    double eps_singular, double *d_centers, double *d_sizes, uint8_t *d_singular);

#ifdef __cplusplus
}
#endif
#endif
