// alphax_b200.cu -- C-ABI entry points (include/alphax_b200.h) and host-side
// orchestration of the CUDA kernels.  One translation unit; compile with
//   nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false -lineinfo ...
// (-fmad=false is part of the contract: see predicates.cuh).
#include "../../include/alphax_b200.h"

#include "canon.cuh"
#include "common.cuh"
#include "edges.cuh"
#include "estimate.cuh"
#include "estimate3.cuh"
#include "grid.cuh"
#include "heavy.cuh"
#include "predicates.cuh"
#include "prune.cuh"
#include "scan.cuh"
#include "sparse.cuh"
#include "stages.cuh"
#include "sweep.cuh"
#include "widen_pool.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <new>
#include <atomic>
#include <thread>
#include <vector>

using namespace axb;

namespace {

constexpr size_t ARENA_ALIGN = 256;
constexpr int64_t MAX_CELLS = (int64_t)1 << 31;   // dense cell table limit (uint32 keys, 8 GiB of table)

struct HostBlock {            // pinned; filled by async copies
    Counters ctr;
    BoundsPartial bounds;
    uint32_t totals[4];
    ErrRecord errs[ERR_CAP];
    int2 dups[DUP_CAP];
};

enum State { S_NONE = 0, S_GRID = 1, S_EDGES = 2, S_POTENTIAL = 3, S_PRUNED = 4, S_CANON = 5 };

}  // namespace

struct axb_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;     // D2H of finished dimensions overlaps the remaining kernels
    cudaEvent_t dim_ready[4] = {}, dim_count[4] = {};
    // host path: rows cross PCIe as int32 into this pinned staging area and are widened by the pool
    int32_t *h_stage = nullptr;
    size_t h_stage_elems = 0;
    char *h_in = nullptr;                   // pinned staging area for pageable inputs
    size_t h_in_bytes = 0;
    axb::WidenPool *pool = nullptr;
    std::vector<cudaEvent_t> chunk_ev;
    int64_t last_d2h_bytes = 0;
    char *arena = nullptr;
    size_t arena_bytes = 0, arena_used = 0, arena_needed = 0;
    HostBlock *h = nullptr;
    HostBlock *h_dev = nullptr;             // device-side address of the same pinned block (zero-copy stores)
    int state = S_NONE;
    int last_status = AXB_OK;
    int64_t err_verts[4] = {-1, -1, -1, -1};
    int err_nverts = 0;
    unsigned long long err_key = 0;         // AXB_ERR_DEGENERATE: the enumeration key of the reported solve
    double err_xyz[3] = {0, 0, 0};          // AXB_ERR_DUPLICATE: the shared centre
    char msg[512] = {0};
    int64_t launches = 0;
    cudaEvent_t ev[AXB_ST_COUNT + 2] = {};      // stage boundaries 0..EXPORT, then export begin/end
    bool ev_set[AXB_ST_COUNT + 2] = {};
    float stage_ms[AXB_ST_COUNT] = {};
    bool stage_timing = false;             // axb_set_stage_timing

    // run
    axb_params prm = {};
    int64_t n = 0;
    const double *d_xyz = nullptr, *d_radii = nullptr;
    axb_grid_info ginfo = {};
    GridView g = {};
    Tol tol = {};
    int rank_lo = 0, rank_hi = 0;
    int gen_lo = 0;                       // first generator whose simplices are built: rank_lo, or 0 for a slab (the lower
                                          // halo's simplices decide the inherited faces of owned simplices)
    // device arrays (arena)
    Counters *ctr = nullptr;
    ErrRecord *errs = nullptr;
    int2 *dups = nullptr;
    int *key_of_ball = nullptr, *orig = nullptr, *rank = nullptr;
    long long *key64_of_ball = nullptr, *skeys = nullptr;    // sparse mode (no dense cell table)
    int4 *cell_of_rank = nullptr;
    uint32_t *cell_start = nullptr;
    Atom *atoms = nullptr;
    Atom *xyzr = nullptr;                   // (x, y, z, reach) per rank: the edge stage's candidate record
    double *reach = nullptr;
    uint32_t *adj_off = nullptr;
    int *deg = nullptr, *pe_u = nullptr, *pe_v = nullptr;
    uint32_t pe_cap = 0, pt_cap = 0, pq_cap = 0, k3_cap = 0;
    int4 *pt = nullptr, *pq_r = nullptr;
    int *pq_l = nullptr;
    int W = 1;
    int *heavy_list = nullptr;              // generators with more than 256 partners (heavy.cuh), when there are any
    unsigned long long *heavy_scratch = nullptr;
    unsigned heavy_blocks = 0;
    unsigned long long *trimask = nullptr;
    unsigned int *eflag = nullptr;
    unsigned char *vflag = nullptr;
    int4 *k3 = nullptr;
    uint32_t *cnt1 = nullptr, *cnt2 = nullptr, *cnt3 = nullptr, *vkeep = nullptr;
    uint32_t *off1 = nullptr, *off2 = nullptr, *off3 = nullptr, *voff = nullptr;
    int2 *tmp1 = nullptr;
    int4 *tmp2 = nullptr, *tmp3 = nullptr;
    uint32_t n_pe = 0, n_pt = 0, n_pq = 0;
    int64_t counts[4] = {0, 0, 0, 0};
    int64_t host_cap[4] = {0, 0, 0, 0};
    size_t mark_after_grid = 0, mark_after_edges = 0, arena_after_prune = 0;
    int cull_mask = 1;                    // bit 0: tets, bit 1: triangles (A/B switch AXB_CULL=0..3)
    bool cull = false;                    // one-call path: k_tri_tet3 settles partner-dominated simplices itself
    bool slab_mode = false;               // grid geometry fixed by the caller (one z-slab of a global grid)
    bool many_tets = false;               // > 20 partner pairs per generator: heavy tile shape, claimed tet chunks
    bool defer_dup = false;               // one-call paths: the duplicate-centre check rides on the edge stage's host sync
    bool dup_pending = false;
    const int64_t *gidx = nullptr;        // slab mode: global ball index per local ball (ascending)
    // alpha sweep (sweep.cuh)
    // What the edge stage found last time, per problem shape: with it the one-call path sizes the lists and picks the kernel
    // shapes WITHOUT waiting for this run's edge counters, and verifies everything at its final sync (edges_assumed)
    struct EdgeMemo {
        bool valid = false;
        int64_t n = 0, dims[3] = {0, 0, 0};
        double alpha = 0, eps_abs = 0, eps_sing = 0;
        int biomolecule = 0;
        uint32_t n_pe = 0;
        unsigned max_deg = 0;
        unsigned long long pair_bound = 0;
    } memo;
    bool edges_assumed = false, allow_assume = false;
    cudaEvent_t side_go = nullptr, side_done = nullptr;     // hand-over to / from the second stream (early memset)
    bool prune_prealloc = false, side_pending = false;
    bool sweep_ready = false, sweep_on = false, sweep_ranked = false;
    bool lists_complete = false;          // the resident potential lists were built without cull mode
    SweepArrays sw = {};
    size_t mark_after_sweep = 0;
};

namespace {

int fail(axb_ctx *c, int status, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
int fail(axb_ctx *c, int status, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->msg, sizeof(c->msg), fmt, ap);
    va_end(ap);
    c->last_status = status;
    return status;
}

#define CUDA_TRY(c, expr)                                                                           \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail((c), AXB_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                        \
    } while (0)

#define LAUNCH_CHECK(c)                                                                                        \
    do {                                                                                                       \
        (c)->launches++;                                                                                       \
        cudaError_t e_ = cudaGetLastError();                                                                   \
        if (e_ != cudaSuccess)                                                                                 \
            return fail((c), AXB_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                                             \
    } while (0)

template <class T>
T *arena_alloc(axb_ctx *c, size_t count) {
    size_t bytes = (count * sizeof(T) + ARENA_ALIGN - 1) / ARENA_ALIGN * ARENA_ALIGN;
    if (bytes == 0) bytes = ARENA_ALIGN;
    size_t want = c->arena_used + bytes;
    if (want > c->arena_needed) c->arena_needed = want;
    if (want > c->arena_bytes || c->arena == nullptr) return nullptr;
    T *p = reinterpret_cast<T *>(c->arena + c->arena_used);
    c->arena_used = want;
    return p;
}

#define ARENA(c, ptr, T, count)                                                                         \
    do {                                                                                                \
        (ptr) = arena_alloc<T>((c), (count));                                                           \
        if (!(ptr))                                                                                     \
            return fail((c), AXB_ERR_ARENA, "scratch arena too small: need at least %zu bytes, have %zu", \
                        (c)->arena_needed, (c)->arena_bytes);                                           \
    } while (0)

inline unsigned blocks_for(size_t items, int threads) { return (unsigned)std::max<size_t>(1, (items + threads - 1) / threads); }

int mark_event(axb_ctx *c, int idx) {
    // only on request (axb_set_stage_timing): ~30 event records per run cost 0.04-0.06 ms of stream and host time
    // (1M atoms: 1.43 -> 1.38 ms per run, 1k atoms: 0.22 -> 0.18 ms)
    if (!c->stage_timing) return AXB_OK;
    CUDA_TRY(c, cudaEventRecord(c->ev[idx], c->stream));
    c->ev_set[idx] = true;
    return AXB_OK;
}

// exclusive scans of up to four equally long uint32 arrays in ONE launch (out has n + 1 entries, may alias in):
// single pass with decoupled look-back (scan.cuh); a few tiles: one block per array walks them with a carry
int device_scan_many(axb_ctx *c, int arrays, const uint32_t *const in[4], size_t n, uint32_t *const out[4]) {
    Scan4 a{};
    for (int k = 0; k < arrays; ++k) { a.in[k] = in[k]; a.out[k] = out[k]; }
    const size_t ntiles = (n + 1 + SCAN_TILE - 1) / SCAN_TILE;
    if (ntiles <= SCAN_SMALL_TILES) {
        k_scan_small<<<arrays, SCAN_THREADS, 0, c->stream>>>(a, n);
        LAUNCH_CHECK(c);
        return AXB_OK;
    }
    unsigned long long *status;
    ARENA(c, status, unsigned long long, (size_t)arrays * ntiles + 1);     // + the four tickets
    for (int k = 0; k < arrays; ++k) a.status[k] = status + (size_t)k * ntiles;
    a.ticket = reinterpret_cast<unsigned int *>(status + (size_t)arrays * ntiles);
    static_assert(sizeof(unsigned long long) * 2 >= sizeof(unsigned int) * 4, "tickets");
    unsigned int *extra;
    ARENA(c, extra, unsigned int, 4);
    (void)extra;                                                           // keeps the tickets inside the allocation
    CUDA_TRY(c, cudaMemsetAsync(status, 0, sizeof(unsigned long long) * ((size_t)arrays * ntiles + 1) + 16, c->stream));
    k_scan_lookback<<<dim3((unsigned)ntiles, (unsigned)arrays), LB_THREADS, 0, c->stream>>>(a, n);
    LAUNCH_CHECK(c);
    return AXB_OK;
}

int device_scan(axb_ctx *c, const uint32_t *in, size_t n, uint32_t *out) {
    const uint32_t *const i4[4] = {in, nullptr, nullptr, nullptr};
    uint32_t *const o4[4] = {out, nullptr, nullptr, nullptr};
    return device_scan_many(c, 1, i4, n, o4);
}

int device_scan4(axb_ctx *c, const uint32_t *const in[4], size_t n, uint32_t *const out[4]) {
    return device_scan_many(c, 4, in, n, out);
}

__global__ void k_publish_state(const uint32_t *__restrict__ t0, const uint32_t *__restrict__ t1, const uint32_t *__restrict__ t2,
                                const uint32_t *__restrict__ t3, const Counters *__restrict__ ctr, uint32_t *h_totals,
                                Counters *h_ctr) {
    const unsigned *src = reinterpret_cast<const unsigned *>(ctr);
    unsigned *dst = reinterpret_cast<unsigned *>(h_ctr);
    for (unsigned w = threadIdx.x; w < sizeof(Counters) / sizeof(unsigned); w += blockDim.x) dst[w] = src[w];
    if (threadIdx.x == 0) { h_totals[0] = *t0; h_totals[1] = *t1; h_totals[2] = *t2; h_totals[3] = *t3; }
    __threadfence_system();
}

int fetch_counters(axb_ctx *c) {
    CUDA_TRY(c, cudaMemcpyAsync(&c->h->ctr, c->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return AXB_OK;
}

// sparse twin of bin_balls: stable radix sort by 64-bit cell key (sparse.cuh)
int bin_balls_sparse(axb_ctx *c, double side, const double lo[3], const int64_t dims[3]) {
    const int n = (int)c->n;
    const int64_t G = dims[0] * dims[1] * dims[2];
    c->ginfo.cell_side = side;
    for (int a = 0; a < 3; ++a) { c->ginfo.origin[a] = lo[a]; c->ginfo.dims[a] = dims[a]; }
    c->ginfo.n_cells = G;
    c->ginfo.n_balls = c->n;
    GridView &g = c->g;
    g.ox = lo[0]; g.oy = lo[1]; g.oz = lo[2];
    g.side = side;
    g.dx = (int)dims[0]; g.dy = (int)dims[1]; g.dz = (int)dims[2];
    g.z_lo = 0;
    g.dz_glob = (int)dims[2];
    g.n = n;
    g.cell_start = nullptr;
    c->cell_start = nullptr;
    c->key_of_ball = nullptr;
    ARENA(c, c->key64_of_ball, long long, n);
    ARENA(c, c->skeys, long long, n);
    ARENA(c, c->orig, int, n);
    ARENA(c, c->rank, int, n);
    ARENA(c, c->cell_of_rank, int4, n);
    ARENA(c, c->atoms, Atom, n);
    ARENA(c, c->reach, double, n);
    ARENA(c, c->xyzr, Atom, n);
    const size_t mark = c->arena_used;
    long long *kbuf;
    int *vbuf[2];
    uint32_t *hist;
    const int nchunks = (n + RS_CHUNK - 1) / RS_CHUNK;
    ARENA(c, kbuf, long long, n);
    ARENA(c, vbuf[0], int, n);
    ARENA(c, vbuf[1], int, n);
    ARENA(c, hist, uint32_t, (size_t)256 * nchunks + 2);
    g.skeys = c->skeys;
    k_cell_keys64<<<blocks_for(n, 256), 256, 0, c->stream>>>(c->d_xyz, g, c->key64_of_ball, c->skeys, vbuf[0]);
    LAUNCH_CHECK(c);
    int bits = 0;
    while (bits < 63 && ((int64_t)1 << bits) < G) ++bits;
    long long *kin = c->skeys, *kout = kbuf;
    int cur = 0;
    const unsigned rs_blocks = (unsigned)((nchunks + RS_WARPS - 1) / RS_WARPS);
    for (int shift = 0; shift < std::max(bits, 1); shift += 8) {
        k_rs_hist<<<rs_blocks, RS_WARPS * 32, 0, c->stream>>>(kin, n, shift, nchunks, hist);
        LAUNCH_CHECK(c);
        int st = device_scan(c, hist, (size_t)256 * nchunks, hist);
        if (st != AXB_OK) return st;
        k_rs_scatter<<<rs_blocks, RS_WARPS * 32, 0, c->stream>>>(kin, vbuf[cur], n, shift, nchunks, hist, kout, vbuf[cur ^ 1]);
        LAUNCH_CHECK(c);
        std::swap(kin, kout);
        cur ^= 1;
    }
    if (kin != c->skeys)
        CUDA_TRY(c, cudaMemcpyAsync(c->skeys, kin, sizeof(long long) * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    k_sparse_finalize<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->d_xyz, c->d_radii, c->skeys, vbuf[cur], g, c->prm.alpha,
                                                               c->prm.eps_abs, c->orig, c->rank, c->cell_of_rank, c->atoms,
                                                               c->reach, c->xyzr, c->ctr, c->dups);
    LAUNCH_CHECK(c);
    c->arena_used = mark;
    return AXB_OK;
}

// counting sort of the balls by cell key + rank-space records (grid.cuh).
// dims = dims of the GLOBAL grid; [z_lo, z_hi) = loaded z layers (the whole grid unless this is a slab).
int bin_balls(axb_ctx *c, double side, const double lo[3], const int64_t dims[3], int64_t z_lo, int64_t z_hi) {
    const int n = (int)c->n;
    const int64_t zc = z_hi - z_lo;
    if (dims[0] >= MAX_CELLS || dims[1] >= MAX_CELLS || dims[2] >= MAX_CELLS)
        return fail(c, AXB_ERR_GRID_TOO_LARGE, "a grid axis of %lld x %lld x %lld cells exceeds 2^31",
                    (long long)dims[0], (long long)dims[1], (long long)dims[2]);
    long double cells = (long double)dims[0] * (long double)dims[1] * (long double)zc;
    if (cells >= 4.0e18L) return fail(c, AXB_ERR_GRID_TOO_LARGE, "cell keys would overflow 63 bits");
    // a dense table pays off while it is not much larger than the input; beyond that (or beyond 2^31 cells)
    // bin by sorting the keys
    const bool force_sparse = getenv("AXB_FORCE_SPARSE") != nullptr;      // test hook
    const bool sparse = force_sparse || cells >= (long double)MAX_CELLS || cells > 64.0L * (long double)n + 16777216.0L;
    if (sparse) {
        if (c->slab_mode) return fail(c, AXB_ERR_GRID_TOO_LARGE, "slab sharding needs the dense cell table");
        return bin_balls_sparse(c, side, lo, dims);
    }
    const int64_t G = dims[0] * dims[1] * zc;
    c->ginfo.cell_side = side;
    for (int a = 0; a < 3; ++a) { c->ginfo.origin[a] = lo[a]; c->ginfo.dims[a] = dims[a]; }
    c->ginfo.n_cells = G;
    c->ginfo.n_balls = c->n;
    GridView &g = c->g;
    g.ox = lo[0]; g.oy = lo[1]; g.oz = lo[2];
    g.side = side;
    g.dx = (int)dims[0]; g.dy = (int)dims[1]; g.dz = (int)zc;
    g.z_lo = (int)z_lo;
    g.dz_glob = (int)dims[2];
    g.n = n;

    uint32_t *cell_count;
    int *arrival;
    ARENA(c, c->key_of_ball, int, n);
    ARENA(c, c->cell_start, uint32_t, (size_t)G + 2);
    ARENA(c, c->orig, int, n);
    ARENA(c, c->rank, int, n);
    ARENA(c, c->cell_of_rank, int4, n);
    ARENA(c, c->atoms, Atom, n);
    ARENA(c, c->reach, double, n);
    ARENA(c, c->xyzr, Atom, n);
    const size_t mark = c->arena_used;          // everything below is scratch of this function
    ARENA(c, cell_count, uint32_t, (size_t)G + 2);
    ARENA(c, arrival, int, n);
    g.cell_start = c->cell_start;
    g.skeys = nullptr;
    c->skeys = nullptr;

    CUDA_TRY(c, cudaMemsetAsync(cell_count, 0, ((size_t)G + 2) * sizeof(uint32_t), c->stream));
    k_cell_keys<<<blocks_for(n, 256), 256, 0, c->stream>>>(c->d_xyz, g, c->key_of_ball, cell_count);
    LAUNCH_CHECK(c);
    int st = device_scan(c, cell_count, (size_t)G + 1, c->cell_start);
    if (st != AXB_OK) return st;
    k_cell_scatter<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->key_of_ball, c->cell_start, cell_count, arrival);
    LAUNCH_CHECK(c);
    k_cell_finalize<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->d_xyz, c->d_radii, c->key_of_ball, c->cell_start,
                                                             arrival, c->prm.alpha, c->prm.eps_abs, c->orig, c->rank,
                                                             c->cell_of_rank, g.dx, g.dy, c->atoms, c->reach, c->xyzr, c->ctr, c->dups);
    LAUNCH_CHECK(c);
    // the scratch is dead once the stream has passed k_cell_finalize; later stages
    // are ordered on the same stream, so it can be handed out again
    c->arena_used = mark;
    return AXB_OK;
}

// slab mode: the kernels name balls by their position in the slab's input; callers know them by global index
int globalize_err_verts(axb_ctx *c) {
    if (!c->gidx) return AXB_OK;
    for (int a = 0; a < c->err_nverts; ++a) {
        int64_t g = -1;
        CUDA_TRY(c, cudaMemcpy(&g, c->gidx + c->err_verts[a], sizeof(int64_t), cudaMemcpyDeviceToHost));
        c->err_verts[a] = g;
    }
    std::sort(c->err_verts, c->err_verts + c->err_nverts);     // gidx ascends, so this keeps the order anyway
    return AXB_OK;
}

// pick the duplicate pair the reference reports (pipeline.py:238-244): first adjacent equal
// pair in lexsort (x, y, z) order == smallest centre, then the two smallest ball indices.
int report_duplicate(axb_ctx *c, unsigned ndup) {
    CUDA_TRY(c, cudaMemcpyAsync(c->h->dups, c->dups, sizeof(int2) * std::min<unsigned>(ndup, DUP_CAP),
                                cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    unsigned m = std::min<unsigned>(ndup, DUP_CAP);
    int best = -1;
    double bx[3] = {0, 0, 0};
    for (unsigned q = 0; q < m; ++q) {
        double p[3];
        CUDA_TRY(c, cudaMemcpy(p, c->d_xyz + 3 * (size_t)c->h->dups[q].x, sizeof(p), cudaMemcpyDeviceToHost));
        bool better = best < 0;
        if (!better) {
            if (p[0] != bx[0]) better = p[0] < bx[0];
            else if (p[1] != bx[1]) better = p[1] < bx[1];
            else if (p[2] != bx[2]) better = p[2] < bx[2];
            else better = c->h->dups[q].x < c->h->dups[best].x;
        }
        if (better) { best = (int)q; bx[0] = p[0]; bx[1] = p[1]; bx[2] = p[2]; }
    }
    c->err_verts[0] = c->h->dups[best].x;
    c->err_verts[1] = c->h->dups[best].y;
    c->err_nverts = 2;
    for (int a = 0; a < 3; ++a) c->err_xyz[a] = bx[a];
    int ms = globalize_err_verts(c);
    if (ms != AXB_OK) return ms;
    return fail(c, AXB_ERR_DUPLICATE, "balls %lld and %lld share the center (%.17g, %.17g, %.17g)",
                (long long)c->err_verts[0], (long long)c->err_verts[1], bx[0], bx[1], bx[2]);
}

EstParams est_params(axb_ctx *c, unsigned long long report_key) {
    EstParams P;
    P.g = c->g; P.tol = c->tol;
    P.atoms = c->atoms; P.xyzr = c->xyzr; P.reach = c->reach; P.orig = c->orig; P.cell_of_rank = c->cell_of_rank;
    P.adj_off = c->adj_off; P.deg = c->deg; P.pe_v = c->pe_v; P.pe_u = c->pe_u; P.pe_cap = c->pe_cap;
    P.pt = c->pt; P.pt_cap = c->pt_cap; P.pq_r = c->pq_r; P.pq_l = c->pq_l; P.pq_cap = c->pq_cap;
    P.ctr = c->ctr; P.errs = c->errs; P.report_key = report_key;
    P.cull = c->cull ? c->cull_mask : 0;
    // a slab reports singular solves only for generators whose enumeration is complete (the upper halo's is not)
    P.err_rank_hi = c->slab_mode ? c->rank_hi : 0x7fffffff;
    P.own_lo = c->slab_mode ? c->rank_lo : 0;
    return P;
}

PruneParams prune_params(axb_ctx *c) {
    PruneParams P;
    P.g = c->g; P.tol = c->tol;
    P.atoms = c->atoms; P.orig = c->orig; P.adj_off = c->adj_off; P.deg = c->deg;
    P.pe_u = c->pe_u; P.pe_v = c->pe_v; P.pt = c->pt; P.pq_r = c->pq_r; P.pq_l = c->pq_l;
    P.pt_cap = c->pt_cap; P.pq_cap = c->pq_cap; P.pe_cap = c->pe_cap;
    P.W = c->W; P.trimask = c->trimask; P.eflag = c->eflag; P.vflag = c->vflag; P.k3 = c->k3;
    P.cnt1 = c->cnt1; P.cnt2 = c->cnt2; P.cnt3 = c->cnt3; P.vkeep = c->vkeep;
    P.ctr = c->ctr; P.biomolecule = c->prm.biomolecule;
    P.rank_lo = c->rank_lo; P.rank_hi = c->rank_hi;
    P.own_only = c->slab_mode ? 1 : 0;
    P.sweep = c->sweep_on ? 1 : 0;
    P.sw_pf = c->sw.pf; P.sw_tsize = c->sw.tsize; P.sw_tvw = c->sw.tvw; P.sw_qsize = c->sw.qsize; P.sw_qtsize = c->sw.qtsize;
    P.sw_qe = c->sw.qe; P.sw_ac2e = c->sw.ac2e; P.sw_ac2t = c->sw.ac2t; P.sw_ac2q = c->sw.ac2q;
    P.k3_cap = c->k3_cap;
    // n_pt may still be the optimistic capacity (axb_compute); the potential triangles are ~0.8 per potential edge
    const unsigned warps = (unsigned)c->sm_count * (unsigned)PRUNE_GRID * (unsigned)PRUNE_WARPS;
    P.claim_tris = prune_claim(std::min<unsigned long long>(c->n_pt, c->n_pe), (unsigned)c->sm_count * (unsigned)PRUNE_GRID * (unsigned)TRIS_WARPS, PRUNE_CLAIM_TRIS);
    P.claim_edges = prune_claim(c->n_pe, warps, PRUNE_CLAIM_EDGES);
    return P;
}

int launch_edges(axb_ctx *c, const EstParams &P, int lo, int hi) {
    const unsigned nblocks = (unsigned)std::max(1, (hi - lo + 32 * EL_WARPS - 1) / (32 * EL_WARPS));
    const size_t smem = sizeof(ELWarp) * EL_WARPS;
    CUDA_TRY(c, cudaFuncSetAttribute(k_edges, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned resident = (unsigned)c->sm_count * (unsigned)EL_MINB;
    const int dyn = nblocks > resident ? 1 : 0;
    if (dyn) CUDA_TRY(c, cudaMemsetAsync(&c->ctr->work_next[0], 0, sizeof(unsigned int), c->stream));     // tile claims
    k_edges<<<std::min(nblocks, resident), EL_WARPS * 32, smem, c->stream>>>(P, lo, hi, dyn);
    LAUNCH_CHECK(c);
    return AXB_OK;
}

int launch_tri_tet(axb_ctx *c, unsigned long long report_key) {
    EstParams P = est_params(c, report_key);
    const int ngen = c->rank_hi - c->gen_lo;
#ifndef TETS_DYN_PAIRS
#define TETS_DYN_PAIRS 25      // more partner pairs per generator than this: k_prune_tets claims chunks (1M atoms, final kernels:
                               // the static loop wins up to alpha 0.6 = 0.50 vs 0.51 ms (0.4: 0.33 vs 0.38), claims from 0.8 = 0.64 vs 0.70 ms)
#endif
#ifndef T3_HEAVY_PAIRS
#define T3_HEAVY_PAIRS 33     // more partner pairs per generator than this: heavy tile shape (1M atoms, final kernels: light wins up
                              // to alpha 0.8 = 1.04 vs 1.11 ms (0.6: 0.82 vs 0.91), a tie at 1.0, heavy at 1.4 = 1.97 vs 2.07 ms;
                              // tools/gpu_alpha_scan.py; ~11 / 23 / 27 / 33 / 45 pairs per generator at alpha 0 / 0.6 / 0.8 / 1.0 / 1.4)
#endif
    {   // warp-autonomous tiles (estimate3.cuh); the tile shape follows the work per generator
        CUDA_TRY(c, cudaMemsetAsync(&c->ctr->tile_next, 0, 2 * sizeof(unsigned int), c->stream));     // tile_next, n_heavy
        auto launch = [&](auto kernel, size_t warp_bytes, int gens, int minb) -> int {
            const size_t smem = warp_bytes * T3_WARPS;
            const unsigned nblocks = (unsigned)std::max(1, (ngen + gens * T3_WARPS - 1) / (gens * T3_WARPS));
            CUDA_TRY(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kernel<<<std::min(nblocks, (unsigned)c->sm_count * (unsigned)minb), T3_WARPS * 32, smem, c->stream>>>(P, c->gen_lo, c->rank_hi);
            return AXB_OK;
        };
        int st;
        const bool heavy = c->h->ctr.pair_bound > (unsigned long long)T3_HEAVY_PAIRS * (unsigned long long)std::max(ngen, 1);   // partner pairs per generator
        c->many_tets = c->h->ctr.pair_bound > (unsigned long long)TETS_DYN_PAIRS * (unsigned long long)std::max(ngen, 1);   // k_prune_tets variant
        if (c->W != 1) st = launch(k_tri_tet3<4, T3_LIGHT>, sizeof(T3Warp<4, T3_LIGHT>), T3Cfg<4, T3_LIGHT>::GENS, 1);
        else if (heavy) st = launch(k_tri_tet3<1, T3_HEAVY>, sizeof(T3Warp<1, T3_HEAVY>), T3Cfg<1, T3_HEAVY>::GENS, T3Cfg<1, T3_HEAVY>::MINB);
#ifndef T3_SMALL_TILES
#define T3_SMALL_TILES 2      // at most this many tiles per resident warp: the spill-free 16-warp shape
#endif
        else if ((unsigned)ngen <= 16u * T3_WARPS * (unsigned)c->sm_count * (unsigned)T3Cfg<1, T3_LIGHT>::MINB * (unsigned)T3_SMALL_TILES)
            st = launch(k_tri_tet3<1, T3_SMALL>, sizeof(T3Warp<1, T3_SMALL>), T3Cfg<1, T3_SMALL>::GENS, T3Cfg<1, T3_SMALL>::MINB);
        else st = launch(k_tri_tet3<1, T3_LIGHT>, sizeof(T3Warp<1, T3_LIGHT>), T3Cfg<1, T3_LIGHT>::GENS, T3Cfg<1, T3_LIGHT>::MINB);
        if (st != AXB_OK) return st;
        LAUNCH_CHECK(c);
        if (c->heavy_list) {        // some generator has more partners than a tile holds: those go through heavy.cuh
            k_list_heavy<<<blocks_for((size_t)std::max(ngen, 1), 256), 256, 0, c->stream>>>(c->gen_lo, c->rank_hi, c->deg, c->heavy_list,
                                                                                          &c->ctr->n_heavy);
            LAUNCH_CHECK(c);
            k_tri_tet_heavy<<<c->heavy_blocks, HEAVY_THREADS, 0, c->stream>>>(P, c->heavy_list, &c->ctr->n_heavy, c->W, c->heavy_scratch);
            LAUNCH_CHECK(c);
        }
        return AXB_OK;
    }
}

// turn the smallest singular key into the reference's DegenerateSimplex report
int report_degenerate(axb_ctx *c) {
    const unsigned long long key = c->h->ctr.err_key;
    unsigned m = std::min<unsigned>(c->h->ctr.err_count, ERR_CAP);
    CUDA_TRY(c, cudaMemcpyAsync(c->h->errs, c->errs, sizeof(ErrRecord) * std::max(1u, m), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const ErrRecord *hit = nullptr;
    for (unsigned q = 0; q < m && !hit; ++q)
        if (c->h->errs[q].key == key) hit = &c->h->errs[q];
    if (!hit) {
        // more singular solves than record slots: replay the stage with only `key` reporting
        const int stage = (int)(key >> 60);
        if (stage == ST_EDGE) {
            EstParams P = est_params(c, key);
            P.pe_cap = 0;    // count only
            const int edge_hi = c->slab_mode ? (int)c->n : c->rank_hi;
            int st = launch_edges(c, P, c->gen_lo, edge_hi);
            if (st != AXB_OK) return st;
        } else {
            uint32_t pt_cap = c->pt_cap, pq_cap = c->pq_cap;
            c->pt_cap = 0; c->pq_cap = 0;
            int st = launch_tri_tet(c, key);
            c->pt_cap = pt_cap; c->pq_cap = pq_cap;
            if (st != AXB_OK) return st;
        }
        CUDA_TRY(c, cudaMemcpyAsync(c->h->errs, c->errs, sizeof(ErrRecord), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        hit = &c->h->errs[0];
    }
    c->err_nverts = hit->nverts;
    for (int a = 0; a < 4; ++a) c->err_verts[a] = a < hit->nverts ? hit->verts[a] : -1;
    c->err_key = key;
    {
        int ms = globalize_err_verts(c);
        if (ms != AXB_OK) return ms;
    }
    static const char *what[] = {"simplex", "edge", "edge", "triangle", "tetrahedron"};
    const int stage = (int)(key >> 60);
    char vs[128];
    int w = 0;
    for (int a = 0; a < c->err_nverts; ++a) w += snprintf(vs + w, sizeof(vs) - w, a ? ", %lld" : "%lld", (long long)c->err_verts[a]);
    return fail(c, AXB_ERR_DEGENERATE, "%s (%s) has affinely dependent centers", what[stage <= 4 ? stage : 0], vs);
}

int check_run_flags(axb_ctx *c) {
    const Counters &k = c->h->ctr;
    if (k.err_key != ~0ull) return report_degenerate(c);
    if (k.overflow & 1u)
        return fail(c, AXB_ERR_DENSITY, "a ball has more than %d potential-edge partners", AXB_MAX_PARTNERS);
    if (k.overflow & (1u << 3))
        return fail(c, AXB_ERR_INTERNAL,
                    "%u inherited faces have no row in their generator's partner list (cell-boundary corner case)",
                    k.lookup_miss);
    if (k.overflow & (1u << 5)) return fail(c, AXB_ERR_INTERNAL, "duplicate simplex inside an owner bucket");
    return AXB_OK;
}

}  // namespace

// ------------------------------------------------------------------ context

extern "C" int axb_version(void) { return 100; }

extern "C" const char *axb_status_name(int s) {
    static const char *names[] = {"AXB_OK", "AXB_ERR_BAD_ARG", "AXB_ERR_CUDA", "AXB_ERR_ARENA", "AXB_ERR_EMPTY",
                                  "AXB_ERR_NONFINITE", "AXB_ERR_DUPLICATE", "AXB_ERR_DEGENERATE", "AXB_ERR_BAD_SIDE",
                                  "AXB_ERR_GRID_TOO_LARGE", "AXB_ERR_DENSITY", "AXB_ERR_STATE", "AXB_ERR_INTERNAL"};
    return (s >= 0 && s <= AXB_ERR_INTERNAL) ? names[s] : "AXB_ERR_UNKNOWN";
}

extern "C" int axb_ctx_create(axb_ctx **out, int device) {
    if (!out) return AXB_ERR_BAD_ARG;
    *out = nullptr;
    axb_ctx *c = new (std::nothrow) axb_ctx();
    if (!c) return AXB_ERR_INTERNAL;
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void **>(&c->h), sizeof(HostBlock), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->h_dev), c->h, 0);
    for (int i = 0; e == cudaSuccess && i < AXB_ST_COUNT + 2; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; e == cudaSuccess && i < 4; ++i) e = cudaEventCreateWithFlags(&c->dim_ready[i], cudaEventDisableTiming);
    for (int i = 0; e == cudaSuccess && i < 4; ++i) e = cudaEventCreateWithFlags(&c->dim_count[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->side_go, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->side_done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        fprintf(stderr, "axb_ctx_create: %s\n", cudaGetErrorString(e));
        delete c;
        return AXB_ERR_CUDA;
    }
    *out = c;
    return AXB_OK;
}

extern "C" void axb_ctx_destroy(axb_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    for (int i = 0; i < AXB_ST_COUNT + 2; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    for (int i = 0; i < 4; ++i) {
        if (c->dim_ready[i]) cudaEventDestroy(c->dim_ready[i]);
        if (c->dim_count[i]) cudaEventDestroy(c->dim_count[i]);
    }
    if (c->side_go) cudaEventDestroy(c->side_go);
    if (c->side_done) cudaEventDestroy(c->side_done);
    delete c->pool;
    for (cudaEvent_t e : c->chunk_ev) cudaEventDestroy(e);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_in) cudaFreeHost(c->h_in);
    if (c->h) cudaFreeHost(c->h);
    delete c;
}

extern "C" int axb_ctx_set_stream(axb_ctx *c, void *s) {
    if (!c) return AXB_ERR_BAD_ARG;
    c->stream = reinterpret_cast<cudaStream_t>(s);
    return AXB_OK;
}

extern "C" int axb_ctx_set_arena(axb_ctx *c, void *p, size_t bytes) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (reinterpret_cast<uintptr_t>(p) % ARENA_ALIGN) return fail(c, AXB_ERR_BAD_ARG, "arena must be %zu-byte aligned", ARENA_ALIGN);
    c->arena = static_cast<char *>(p);
    c->arena_bytes = bytes;
    c->arena_used = 0;
    c->arena_needed = 0;
    c->state = S_NONE;
    return AXB_OK;
}

extern "C" size_t axb_arena_needed(const axb_ctx *c) { return c ? c->arena_needed : 0; }
extern "C" size_t axb_arena_used(const axb_ctx *c) { return c ? c->arena_used : 0; }

extern "C" size_t axb_arena_hint(int64_t n, double alpha, double r_max) {
    // ~ one cell per ball at protein density plus the per-simplex lists; alpha widens everything
    double widen = 1.0;
    if (r_max > 0.0 && alpha > 0.0) widen = pow(1.0 + alpha / (r_max * r_max), 1.5);
    double per_atom = 900.0 + 1400.0 * widen * widen;
    double bytes = 64.0 * 1024 * 1024 + per_atom * (double)(n > 0 ? n : 1);
    return (size_t)bytes;
}

extern "C" const char *axb_last_message(const axb_ctx *c) { return c ? c->msg : "null context"; }

extern "C" int axb_last_error(const axb_ctx *c, int *status, int64_t verts[4], int *nverts) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (status) *status = c->last_status;
    if (verts) for (int a = 0; a < 4; ++a) verts[a] = c->err_verts[a];
    if (nverts) *nverts = c->err_nverts;
    return AXB_OK;
}

extern "C" int axb_last_error_detail(const axb_ctx *c, uint64_t *key, double xyz[3]) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (key) *key = c->err_key;
    if (xyz) for (int a = 0; a < 3; ++a) xyz[a] = c->err_xyz[a];
    return AXB_OK;
}

extern "C" int64_t axb_kernel_launches(const axb_ctx *c) { return c ? c->launches : 0; }

extern "C" int axb_set_stage_timing(axb_ctx *c, int on) {
    if (!c) return AXB_ERR_BAD_ARG;
    c->stage_timing = on != 0;
    return AXB_OK;
}

extern "C" int axb_stage_ms(const axb_ctx *cc, float out[AXB_ST_COUNT]) {
    axb_ctx *c = const_cast<axb_ctx *>(cc);
    if (!c || !out) return AXB_ERR_BAD_ARG;
    for (int i = 0; i < AXB_ST_COUNT; ++i) {
        out[i] = 0.f;
        // stages 0..CANONICAL are delimited by ev[i], ev[i+1]; EXPORT by its own pair
        const int a = i == AXB_ST_EXPORT ? AXB_ST_COUNT : i, b = a + 1;
        if (c->ev_set[a] && c->ev_set[b]) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) == cudaSuccess) out[i] = ms;
        }
    }
    return AXB_OK;
}

// --------------------------------------------------------------------- grid

namespace {

// shared body of axb_grid_build / axb_grid_build_slab
int grid_build_common(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *prm,
                      const axb_slab *slab, const int64_t *d_gidx) {
    if (!c || !prm) return AXB_ERR_BAD_ARG;
    c->state = S_NONE;
    c->last_status = AXB_OK;
    c->msg[0] = 0;
    c->err_nverts = 0;
    c->err_key = 0;
    for (int a = 0; a < 4; ++a) c->err_verts[a] = -1;
    for (int i = 0; i < AXB_ST_COUNT + 2; ++i) c->ev_set[i] = false;
    c->arena_used = 0;
    c->arena_needed = 0;
    c->slab_mode = slab != nullptr;
    c->gidx = d_gidx;
    c->sweep_ready = false;
    c->sweep_on = false;
    c->sweep_ranked = false;
    c->prune_prealloc = false;
    c->side_pending = false;
    if (n <= 0) return fail(c, AXB_ERR_EMPTY, "at least one ball is required");
    if (n >= ((int64_t)1 << 31) - 1) return fail(c, AXB_ERR_BAD_ARG, "more than 2^31 - 2 balls are not supported");
    if (!d_xyz || !d_radii) return fail(c, AXB_ERR_BAD_ARG, "null input pointer");
    if (!(prm->eps_abs > 0.0) || !(prm->eps_singular > 0.0) || !isfinite(prm->alpha))
        return fail(c, AXB_ERR_BAD_ARG, "alpha must be finite and tolerances strictly positive");
    if (slab && (!(slab->cell_side > 0.0) || slab->dims[0] < 1 || slab->dims[1] < 1 || slab->dims[2] < 1 ||
                 slab->z_lo < 0 || slab->z_hi > slab->dims[2] || slab->z_lo >= slab->z_hi))
        return fail(c, AXB_ERR_BAD_ARG, "bad slab geometry");
    CUDA_TRY(c, cudaSetDevice(c->device));
    c->prm = *prm;
    c->n = n;
    c->d_xyz = d_xyz;
    c->d_radii = d_radii;
    c->tol.eps_abs = prm->eps_abs;
    c->tol.eps_sing = prm->eps_singular;
    c->tol.lim_a = prm->alpha + prm->eps_abs;

    int st = mark_event(c, AXB_ST_GRID);
    if (st != AXB_OK) return st;
    ARENA(c, c->ctr, Counters, 1);
    ARENA(c, c->errs, ErrRecord, ERR_CAP);
    ARENA(c, c->dups, int2, DUP_CAP);
    const unsigned nb = std::max(1u, std::min(blocks_for((size_t)n, BOUNDS_THREADS * 4), (unsigned)c->sm_count * 8u));
    BoundsPartial *partials, *bres;
    unsigned int *done;
    ARENA(c, partials, BoundsPartial, nb);
    ARENA(c, bres, BoundsPartial, 1);
    ARENA(c, done, unsigned int, 1);
    memset(&c->h->ctr, 0, sizeof(Counters));
    c->h->ctr.err_key = ~0ull;
    c->h->ctr.first_bad = 0xffffffffu;
    CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(done, 0, sizeof(unsigned int), c->stream));
    // the folded result goes straight into mapped host memory (no copy operation between the kernel and the sync)
    (void)bres;
    k_bounds<<<nb, BOUNDS_THREADS, 0, c->stream>>>(d_xyz, d_radii, (int)n, partials, done, &c->h_dev->bounds);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const BoundsPartial &b = c->h->bounds;
    c->tol.r2max = b.rmax * b.rmax;
    c->tol.reach_max = sqrt(std::max(c->tol.r2max + prm->alpha + prm->eps_abs, 0.0)) * (1.0 + 1e-12);
    if (b.first_bad != 0xffffffffu) {                     // pipeline.py:235-237
        c->err_verts[0] = b.first_bad;
        c->err_nverts = 1;
        return fail(c, AXB_ERR_NONFINITE, "ball %u is not finite", b.first_bad);
    }
    bool bad_side = false;
    if (slab) {
        st = bin_balls(c, slab->cell_side, slab->origin, slab->dims, slab->z_lo, slab->z_hi);
    } else {
        const double side_sq = b.rmax * b.rmax + prm->alpha;   // grid.py:112-113
        bad_side = !(side_sq > 0.0);
        double side = bad_side ? 0.0 : sqrt(side_sq);          // grid.py:118
        if (bad_side) {
            // the reference validates duplicates BEFORE it looks at the cell side (pipeline.py:583 then 594),
            // so bin with a stand-in side just to find them
            double span = std::max(b.hi[0] - b.lo[0], std::max(b.hi[1] - b.lo[1], b.hi[2] - b.lo[2]));
            side = span > 0.0 ? span / 128.0 : 1.0;
        }
        int64_t dims[3];
        for (int a = 0; a < 3; ++a) {
            double q = floor((b.hi[a] - b.lo[a]) / side) + 1.0;   // grid.py:121
            if (!(q < 9.0e18)) return fail(c, AXB_ERR_GRID_TOO_LARGE, "grid dimension overflows");
            dims[a] = (int64_t)q;
        }
        st = bin_balls(c, side, b.lo, dims, 0, dims[2]);
    }
    if (st != AXB_OK) return st;
    c->dup_pending = c->defer_dup && !bad_side;
    if (!c->dup_pending) {
        st = fetch_counters(c);
        if (st != AXB_OK) return st;
        if (c->h->ctr.dup_count) return report_duplicate(c, c->h->ctr.dup_count);
    }
    if (bad_side)
        return fail(c, AXB_ERR_BAD_SIDE, "alpha=%.17g gives non-positive squared cell side (r_max=%.17g)", prm->alpha, b.rmax);
    st = mark_event(c, AXB_ST_GRID + 1);
    if (st != AXB_OK) return st;
    c->mark_after_grid = c->arena_used;
    c->state = S_GRID;
    return AXB_OK;
}

}  // namespace

extern "C" int axb_grid_build(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *prm) {
    return grid_build_common(c, n, d_xyz, d_radii, prm, nullptr, nullptr);
}

extern "C" int axb_grid_build_slab(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii,
                                   const int64_t *d_global_index, const axb_params *prm, const axb_slab *slab) {
    if (!slab) return AXB_ERR_BAD_ARG;
    return grid_build_common(c, n, d_xyz, d_radii, prm, slab, d_global_index);
}

extern "C" int axb_slab_rank_range(axb_ctx *c, int64_t z_own_lo, int64_t z_own_hi, int64_t *rank_lo, int64_t *rank_hi) {
    if (!c || !rank_lo || !rank_hi) return AXB_ERR_BAD_ARG;
    if (c->state < S_GRID) return fail(c, AXB_ERR_STATE, "axb_slab_rank_range before axb_grid_build");
    if (!c->cell_start) return fail(c, AXB_ERR_STATE, "axb_slab_rank_range needs the dense cell table");
    const GridView &g = c->g;
    int64_t a = std::min<int64_t>(std::max<int64_t>(z_own_lo - g.z_lo, 0), g.dz);
    int64_t b = std::min<int64_t>(std::max<int64_t>(z_own_hi - g.z_lo, 0), g.dz);
    uint32_t v[2];
    const size_t layer = (size_t)g.dx * g.dy;
    CUDA_TRY(c, cudaMemcpyAsync(&v[0], c->cell_start + layer * (size_t)a, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&v[1], c->cell_start + layer * (size_t)b, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    *rank_lo = v[0];
    *rank_hi = v[1];
    return AXB_OK;
}

extern "C" int axb_grid_get_info(const axb_ctx *c, axb_grid_info *out) {
    if (!c || !out) return AXB_ERR_BAD_ARG;
    if (c->state < S_GRID) return AXB_ERR_STATE;
    *out = c->ginfo;
    return AXB_OK;
}

extern "C" int axb_grid_export(axb_ctx *c, int64_t *d_order, int64_t *d_rank, int64_t *d_cells) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (c->state < S_GRID) return fail(c, AXB_ERR_STATE, "axb_grid_export before axb_grid_build");
    if (c->skeys)
        k_grid_export64<<<blocks_for((size_t)c->n, 256), 256, 0, c->stream>>>((int)c->n, c->orig, c->rank, c->key64_of_ball,
                                                                             d_order, d_rank, d_cells);
    else
        k_grid_export<<<blocks_for((size_t)c->n, 256), 256, 0, c->stream>>>((int)c->n, c->orig, c->rank, c->key_of_ball,
                                                                           d_order, d_rank, d_cells);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return AXB_OK;
}

// ---------------------------------------------------------------- potential

namespace {

// 64-bit words per row of the kept-triangle mask: one up to 64 partners per generator, four up to 256 (the two
// shapes k_tri_tet3 is built for), then as many as the longest partner list needs
int trimask_words(unsigned max_deg) { return max_deg <= 64 ? 1 : (max_deg <= 256 ? 4 : (int)((max_deg + 63) / 64)); }

// list + bit-matrix scratch of the heavy-generator kernel (heavy.cuh), only when some generator needs it
int alloc_heavy(axb_ctx *c) {
    c->heavy_list = nullptr;
    c->heavy_scratch = nullptr;
    if (c->h->ctr.max_deg < (unsigned)HEAVY_MIN_DEG) return AXB_OK;
    c->heavy_blocks = (unsigned)c->sm_count * 2u;
    ARENA(c, c->heavy_list, int, (size_t)c->n + 1);
    ARENA(c, c->heavy_scratch, unsigned long long, (size_t)c->heavy_blocks * 2 * (MAXP + 1) * (size_t)c->W);
    return AXB_OK;
}

// potential edges for generators [lo, hi) (+ the upper halo rows of a slab); synchronises once
int run_edges(axb_ctx *c, int64_t lo, int64_t hi) {
    if (c->state < S_GRID) return fail(c, AXB_ERR_STATE, "axb_potential before axb_grid_build");
    if (lo < 0 || hi > c->n || lo > hi) return fail(c, AXB_ERR_BAD_ARG, "bad rank range");
    c->state = S_GRID;
    c->arena_used = c->mark_after_grid;
    c->rank_lo = (int)lo;
    c->rank_hi = (int)hi;
    c->gen_lo = c->slab_mode ? 0 : (int)lo;
    const int n = (int)c->n;
    const int ngen = (int)(hi - lo);
    int st;
    memset(&c->h->ctr, 0, sizeof(Counters));
    c->h->ctr.err_key = ~0ull;
    c->h->ctr.first_bad = 0xffffffffu;
    // (with a pending duplicate check the device counters are still the grid stage's: all zero but dup_count)
    if (!c->dup_pending)
        CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
    if ((st = mark_event(c, AXB_ST_POT_EDGES)) != AXB_OK) return st;
    ARENA(c, c->adj_off, uint32_t, n);
    ARENA(c, c->deg, int, n);
    const size_t mark_pe = c->arena_used;
    uint64_t want = (uint64_t)16 * (uint64_t)(c->slab_mode ? n : ngen) + 4096;
    c->edges_assumed = false;
    {   // the same problem shape as last time (another frame, the next step of a sweep or a benchmark): no round trip
        const axb_ctx::EdgeMemo &m = c->memo;
        const bool same = c->allow_assume && m.valid && !c->slab_mode && lo == 0 && hi == c->n && m.n == c->n &&
                          m.alpha == c->prm.alpha && m.eps_abs == c->prm.eps_abs && m.eps_sing == c->prm.eps_singular &&
                          m.biomolecule == c->prm.biomolecule && m.dims[0] == c->ginfo.dims[0] && m.dims[1] == c->ginfo.dims[1] &&
                          m.dims[2] == c->ginfo.dims[2] && m.max_deg + 8 <= 64;       // (one-word masks with room to grow)
        if (same && !getenv("AXB_NO_MEMO")) {
            c->pe_cap = m.n_pe + m.n_pe / 32 + 4096;
            ARENA(c, c->pe_v, int, c->pe_cap);
            ARENA(c, c->pe_u, int, c->pe_cap);
            CUDA_TRY(c, cudaMemsetAsync(c->deg, 0, sizeof(int) * (size_t)n, c->stream));
            EstParams P = est_params(c, 0);
            if ((st = launch_edges(c, P, c->gen_lo, c->rank_hi)) != AXB_OK) return st;
            if ((st = mark_event(c, AXB_ST_POT_EDGES + 1)) != AXB_OK) return st;
            c->edges_assumed = true;
            c->n_pe = c->pe_cap;                                        // upper bound until the final sync
            c->h->ctr.pair_bound = m.pair_bound + m.pair_bound / 32 + 4096;   // sizes the triangle / tet lists, picks tile shapes
            c->h->ctr.max_deg = m.max_deg;
            c->W = 1;
            c->heavy_list = nullptr;
            c->heavy_scratch = nullptr;
            c->mark_after_edges = c->arena_used;
            c->state = S_EDGES;
            return AXB_OK;
        }
    }
    for (int attempt = 0;; ++attempt) {
        if (want > 0xfffffff0ull) return fail(c, AXB_ERR_DENSITY, "more than 2^32 potential edges");
        c->arena_used = mark_pe;
        c->pe_cap = (uint32_t)want;
        ARENA(c, c->pe_v, int, c->pe_cap);
        ARENA(c, c->pe_u, int, c->pe_cap);
        CUDA_TRY(c, cudaMemsetAsync(c->deg, 0, sizeof(int) * (size_t)n, c->stream));
        if (attempt) {   // reset the counters the first attempt touched
            c->h->ctr.n_pe = 0; c->h->ctr.max_deg = 0; c->h->ctr.pair_bound = 0; c->h->ctr.overflow = 0; c->h->ctr.n_heavy = 0;
            c->h->ctr.err_key = ~0ull; c->h->ctr.err_count = 0;
            CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
        }
        EstParams P = est_params(c, 0);
        // a slab builds the partner rows of every loaded ball: the lower halo's generate the simplices that decide the
        // inherited faces of owned simplices, the upper halo's receive the marks of owned tets
        const int edge_hi = c->slab_mode ? n : c->rank_hi;
        st = launch_edges(c, P, c->gen_lo, edge_hi);
        if (st != AXB_OK) return st;
        st = fetch_counters(c);
        if (st != AXB_OK) return st;
        if (c->h->ctr.n_heavy) {            // generators with more partners than the pair queue holds (edges.cuh)
            const size_t smem = sizeof(ELWarp) * EL_WARPS;
            CUDA_TRY(c, cudaFuncSetAttribute(k_edges_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_edges_heavy<<<(unsigned)c->sm_count * 2u, EL_WARPS * 32, smem, c->stream>>>(P, c->gen_lo, edge_hi);
            LAUNCH_CHECK(c);
            if ((st = fetch_counters(c)) != AXB_OK) return st;
        }
        if (c->dup_pending) {              // pipeline.py:238-244 comes before any edge is looked at
            c->dup_pending = false;
            if (c->h->ctr.dup_count) return report_duplicate(c, c->h->ctr.dup_count);
        }
        if (c->h->ctr.n_pe <= c->pe_cap) break;
        if (attempt >= 2) return fail(c, AXB_ERR_INTERNAL, "potential-edge buffer still too small after resize");
        want = (uint64_t)c->h->ctr.n_pe + 1024;
    }
    st = mark_event(c, AXB_ST_POT_EDGES + 1);
    if (st != AXB_OK) return st;
    // singular edges are raised before any triangle is looked at (pipeline.py:357)
    st = check_run_flags(c);
    if (st != AXB_OK) return st;
    c->n_pe = c->h->ctr.n_pe;
    c->W = trimask_words(c->h->ctr.max_deg);
    if ((st = alloc_heavy(c)) != AXB_OK) return st;
    c->mark_after_edges = c->arena_used;
    c->state = S_EDGES;
    return AXB_OK;
}

int alloc_prune_arrays(axb_ctx *c, bool early);

// potential triangles + tets into global lists (the standalone stage path); synchronises
// optimistic = true (axb_compute): no host round trip after the kernel; the list sizes are a guess that almost
// always holds, the pruning kernels check it on the device (lists_overflowed) and run_canonicalize reports it, upon
// which the caller redoes the stage with optimistic = false (exact sizes, one sync)
int run_tri_tet_lists(axb_ctx *c, bool optimistic = false, bool redo = false) {
    int st;
    c->lists_complete = !c->cull;
    uint64_t pt_want = c->h->ctr.pair_bound + 32;           // every potential triangle is a partner pair
    uint64_t pq_want = c->h->ctr.pair_bound + 4096;         // first guess; re-run on overflow
    if (!redo && getenv("AXB_TEST_SMALL_PQ")) pq_want = 64;   // test hook: make the first guess fail
    if (redo) {                                             // the counters of the failed optimistic run are on the host
        pq_want = std::max<uint64_t>(pq_want, (uint64_t)c->h->ctr.n_pq + 1024);
        pt_want = std::max<uint64_t>(pt_want, (uint64_t)c->h->ctr.n_pt + 32);
    }
    for (int attempt = redo ? 1 : 0;; ++attempt) {
        if (pt_want > 0xfffffff0ull || pq_want > 0xfffffff0ull)
            return fail(c, AXB_ERR_DENSITY, "more than 2^32 potential triangles or tetrahedra");
        c->arena_used = c->mark_after_edges;
        c->pt_cap = (uint32_t)pt_want;
        c->pq_cap = (uint32_t)pq_want;
        ARENA(c, c->pt, int4, c->pt_cap);
        ARENA(c, c->pq_r, int4, c->pq_cap);
        ARENA(c, c->pq_l, int, c->pq_cap);
        if (attempt) {
            c->h->ctr.n_pt = 0; c->h->ctr.n_pq = 0; c->h->ctr.overflow = 0;
            c->h->ctr.err_key = ~0ull; c->h->ctr.err_count = 0;
            CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
        }
        if (optimistic && attempt == 0) {
            // the pruning state sits behind the lists; its size only needs the edge count and the list capacities
            c->k3_cap = c->pq_cap;
            const size_t keep = c->arena_used;
            if ((st = alloc_prune_arrays(c, /*early=*/true)) != AXB_OK) return st;
            c->arena_after_prune = c->arena_used;
            c->arena_used = keep;
        }
        st = launch_tri_tet(c, 0);
        if (st != AXB_OK) return st;
        if (optimistic && attempt == 0) {
            if ((st = mark_event(c, AXB_ST_POT_TRIANGLES + 1)) != AXB_OK) return st;
            if ((st = mark_event(c, AXB_ST_POT_TETS + 1)) != AXB_OK) return st;
            c->n_pt = c->pt_cap;                            // upper bounds until run_canonicalize reads the counters
            c->n_pq = c->many_tets ? c->pq_cap : 0;         // only its size class matters (k_prune_tets variant)
            c->k3_cap = c->pq_cap;
            c->state = S_POTENTIAL;
            return AXB_OK;
        }
        st = fetch_counters(c);
        if (st != AXB_OK) return st;
        if (c->h->ctr.n_pq <= c->pq_cap && c->h->ctr.n_pt <= c->pt_cap) break;
        if (attempt >= 3) return fail(c, AXB_ERR_INTERNAL, "potential-tet buffer still too small after resize");
        pq_want = (uint64_t)c->h->ctr.n_pq + 1024;
        pt_want = std::max<uint64_t>(pt_want, (uint64_t)c->h->ctr.n_pt + 32);
    }
    if ((st = mark_event(c, AXB_ST_POT_TRIANGLES + 1)) != AXB_OK) return st;
    if ((st = mark_event(c, AXB_ST_POT_TETS + 1)) != AXB_OK) return st;     // one kernel does both
    if ((st = check_run_flags(c)) != AXB_OK) return st;
    c->n_pt = c->h->ctr.n_pt;
    c->n_pq = c->h->ctr.n_pq;
    c->k3_cap = c->pq_cap;
    c->state = S_POTENTIAL;
    return AXB_OK;
}

int run_potential(axb_ctx *c, int64_t lo, int64_t hi, bool optimistic = false) {
    int st = run_edges(c, lo, hi);
    if (st != AXB_OK) return st;
    return run_tri_tet_lists(c, optimistic);
}

// kept-simplex state of the pruning stage (prune.cuh), zeroed
// early = true (axb_compute): called BEFORE k_tri_tet3 is queued; the big memset then runs on the second stream beside that
// kernel (which uses a few per cent of the DRAM bandwidth) instead of in front of the pruning kernels
int alloc_prune_arrays(axb_ctx *c, bool early) {
    if (c->prune_prealloc) { c->prune_prealloc = false; return AXB_OK; }      // done early for this run
    const int n = (int)c->n;
    const size_t rows = (size_t)std::max<uint32_t>(c->n_pe, 1);
    ARENA(c, c->k3, int4, std::max<uint32_t>(c->k3_cap, 1));
    // the zero-initialised arrays are carved back to back, so ONE memset clears them (nine tiny memsets cost
    // ~20 us of stream time between the potential and the pruning stage)
    const size_t zero_from = c->arena_used;
    ARENA(c, c->trimask, unsigned long long, rows * c->W);
    ARENA(c, c->eflag, unsigned int, rows);
    ARENA(c, c->vflag, unsigned char, n);
    ARENA(c, c->cnt1, uint32_t, (size_t)n + 1);
    ARENA(c, c->cnt2, uint32_t, (size_t)n + 1);
    ARENA(c, c->cnt3, uint32_t, (size_t)n + 1);
    ARENA(c, c->vkeep, uint32_t, (size_t)n + 1);
    if (early) {
        // everything queued so far (previous users of this part of the arena included) comes first
        CUDA_TRY(c, cudaEventRecord(c->side_go, c->stream));
        CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->side_go, 0));
        CUDA_TRY(c, cudaMemsetAsync(c->arena + zero_from, 0, c->arena_used - zero_from, c->copy_stream));
        CUDA_TRY(c, cudaEventRecord(c->side_done, c->copy_stream));
        c->prune_prealloc = true;
        c->side_pending = true;
    } else {
        CUDA_TRY(c, cudaMemsetAsync(c->arena + zero_from, 0, c->arena_used - zero_from, c->stream));
    }
    CUDA_TRY(c, cudaMemsetAsync(&c->ctr->n_k3, 0, sizeof(unsigned int) * PRUNE_COUNTER_WORDS, c->stream));
    return AXB_OK;
}

// triangles, edges, vertices of the pruning stage (the tets are done by the caller)
int run_prune_lower(axb_ctx *c) {
    PruneParams P = prune_params(c);
    int st;
    k_prune_tris<<<(unsigned)c->sm_count * (unsigned)PRUNE_GRID, TRIS_THREADS, 0, c->stream>>>(P);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_TRIANGLES + 1)) != AXB_OK) return st;
    k_prune_edges<<<(unsigned)c->sm_count * (unsigned)PRUNE_GRID, PRUNE_THREADS, 0, c->stream>>>(P);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_EDGES + 1)) != AXB_OK) return st;
    k_prune_vertices<<<blocks_for((size_t)c->n, 256), 256, 0, c->stream>>>(P, c->rank_lo, c->rank_hi);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_VERTICES + 1)) != AXB_OK) return st;
    c->state = S_PRUNED;
    return AXB_OK;
}

int run_prune(axb_ctx *c) {
    if (c->state < S_POTENTIAL) return fail(c, AXB_ERR_STATE, "axb_prune before axb_potential");
    if (c->prune_prealloc) c->arena_used = c->arena_after_prune;
    int st = alloc_prune_arrays(c, false);
    if (st != AXB_OK) return st;
    if (c->side_pending) {
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->side_done, 0));
        c->side_pending = false;
    }
    PruneParams P = prune_params(c);
    // few tets per thread: static grid-stride; many (large alpha, dense cores): dynamic 64-tet claims
    if ((uint64_t)c->n_pq > (uint64_t)c->n + c->n / 2)
        k_prune_tets<1><<<(unsigned)c->sm_count * (unsigned)TETS_MINB, 256, 0, c->stream>>>(P);
    else
        k_prune_tets<0><<<(unsigned)c->sm_count * (unsigned)TETS_GRID, 256, 0, c->stream>>>(P);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_TETS + 1)) != AXB_OK) return st;
    return run_prune_lower(c);
}

// After the final sync of a run whose edge stage was not waited for: did the remembered sizes hold?  AXB_OK, an error
// the reference raises before any triangle (duplicate centre), or the sentinel AXB_ERR_ARENA + 1001 (redo, exactly)
int verify_assumed_edges(axb_ctx *c) {
    if (!c->edges_assumed) return AXB_OK;
    const Counters &k = c->h->ctr;
    if (c->dup_pending) {
        c->dup_pending = false;
        if (k.dup_count) return report_duplicate(c, k.dup_count);
    }
    if ((k.overflow & (1u << 4)) || k.n_pe > c->pe_cap || k.max_deg > 64u || k.n_heavy) return AXB_ERR_ARENA + 1001;
    return AXB_OK;
}

// what the next run with this problem shape may assume
void remember_edges(axb_ctx *c) {
    axb_ctx::EdgeMemo &m = c->memo;
    m.valid = !c->slab_mode && c->rank_lo == 0 && c->rank_hi == (int)c->n;
    m.n = c->n;
    for (int a = 0; a < 3; ++a) m.dims[a] = c->ginfo.dims[a];
    m.alpha = c->prm.alpha; m.eps_abs = c->prm.eps_abs; m.eps_sing = c->prm.eps_singular; m.biomolecule = c->prm.biomolecule;
    m.n_pe = c->h->ctr.n_pe; m.max_deg = c->h->ctr.max_deg; m.pair_bound = c->h->ctr.pair_bound;
}

int run_canonicalize(axb_ctx *c, int64_t counts[4]) {
    if (c->state < S_PRUNED) return fail(c, AXB_ERR_STATE, "axb_canonicalize before axb_prune");
    const size_t n = (size_t)c->n;
    int st;
    ARENA(c, c->off1, uint32_t, n + 2);
    ARENA(c, c->off2, uint32_t, n + 2);
    ARENA(c, c->off3, uint32_t, n + 2);
    ARENA(c, c->voff, uint32_t, n + 2);
    {
        const uint32_t *const in[4] = {c->cnt1, c->cnt2, c->cnt3, c->vkeep};
        uint32_t *const out[4] = {c->off1, c->off2, c->off3, c->voff};
        if ((st = device_scan4(c, in, n, out)) != AXB_OK) return st;
    }
    // the four totals and the counter block reach the host as zero-copy stores of ONE small kernel (five copy
    // operations cost ~10 us of stream time before the sync)
    k_publish_state<<<1, 32, 0, c->stream>>>(c->voff + n, c->off1 + n, c->off2 + n, c->off3 + n, c->ctr, c->h_dev->totals,
                                             &c->h_dev->ctr);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if ((st = verify_assumed_edges(c)) != AXB_OK) return st;
    // deferred checks of the optimistic potential stage
    if (c->h->ctr.n_pq > c->pq_cap || c->h->ctr.n_pt > c->pt_cap || c->h->ctr.n_k3 > c->k3_cap)
        return AXB_ERR_ARENA + 1000;                       // sentinel: a guessed buffer was too small, caller re-runs
    if ((st = check_run_flags(c)) != AXB_OK) return st;
    c->n_pe = c->h->ctr.n_pe;
    c->n_pt = c->h->ctr.n_pt;
    c->n_pq = c->h->ctr.n_pq;
    for (int d = 0; d < 4; ++d) c->counts[d] = c->h->totals[d];
    ARENA(c, c->tmp1, int2, std::max<int64_t>(c->counts[1], 1));
    ARENA(c, c->tmp2, int4, std::max<int64_t>(c->counts[2], 1));
    ARENA(c, c->tmp3, int4, std::max<int64_t>(c->counts[3], 1));
    CanonParams P;
    P.n = (int)n; P.orig = c->orig; P.adj_off = c->adj_off; P.pe_u = c->pe_u; P.pe_v = c->pe_v; P.pe_cap = c->pe_cap;
    P.W = c->W; P.trimask = c->trimask; P.eflag = c->eflag; P.k3 = c->k3;
    P.cnt1 = c->cnt1; P.cnt2 = c->cnt2; P.cnt3 = c->cnt3; P.off1 = c->off1; P.off2 = c->off2; P.off3 = c->off3;
    P.tmp1 = c->tmp1; P.tmp2 = c->tmp2; P.tmp3 = c->tmp3; P.ctr = c->ctr;
    P.own_lo = c->slab_mode ? c->rank_lo : 0; P.own_hi = c->slab_mode ? c->rank_hi : 0x7fffffff;
    const unsigned grid = (unsigned)c->sm_count * 8u;
    k_scatter_edges_tris<<<grid, 256, 0, c->stream>>>(P, 0xffffffffu, 0xffffffffu);
    LAUNCH_CHECK(c);
    k_scatter_tets<<<grid, 256, 0, c->stream>>>(P, c->k3_cap, 0xffffffffu);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_CANONICAL + 1)) != AXB_OK) return st;
    if (counts) for (int d = 0; d < 4; ++d) counts[d] = c->counts[d];
    c->state = S_CANON;
    return AXB_OK;
}

// The same, and the four int64 lists straight into caller buffers of the given capacities, with NO host round trip in
// between: buckets and emit kernels take their sizes from the device (clamped to the capacities), one sync at the very
// end reads the totals and the flags.  A capacity that did not hold: sentinel AXB_ERR_ARENA + 1002 (nothing is valid).
int run_canonicalize_into(axb_ctx *c, int64_t counts[4], int64_t *const d_out[4], const int64_t cap[4]) {
    if (c->state < S_PRUNED) return fail(c, AXB_ERR_STATE, "axb_canonicalize before axb_prune");
    const size_t n = (size_t)c->n;
    int st;
    ARENA(c, c->off1, uint32_t, n + 2);
    ARENA(c, c->off2, uint32_t, n + 2);
    ARENA(c, c->off3, uint32_t, n + 2);
    ARENA(c, c->voff, uint32_t, n + 2);
    {
        const uint32_t *const in[4] = {c->cnt1, c->cnt2, c->cnt3, c->vkeep};
        uint32_t *const out[4] = {c->off1, c->off2, c->off3, c->voff};
        if ((st = device_scan4(c, in, n, out)) != AXB_OK) return st;
    }
    unsigned ucap[4];
    for (int d = 0; d < 4; ++d) ucap[d] = (unsigned)std::min<int64_t>(std::max<int64_t>(cap[d], 0), 0xfffffff0ll);
    ARENA(c, c->tmp1, int2, std::max(ucap[1], 1u));
    ARENA(c, c->tmp2, int4, std::max(ucap[2], 1u));
    ARENA(c, c->tmp3, int4, std::max(ucap[3], 1u));
    CanonParams P;
    P.n = (int)n; P.orig = c->orig; P.adj_off = c->adj_off; P.pe_u = c->pe_u; P.pe_v = c->pe_v; P.pe_cap = c->pe_cap;
    P.W = c->W; P.trimask = c->trimask; P.eflag = c->eflag; P.k3 = c->k3;
    P.cnt1 = c->cnt1; P.cnt2 = c->cnt2; P.cnt3 = c->cnt3; P.off1 = c->off1; P.off2 = c->off2; P.off3 = c->off3;
    P.tmp1 = c->tmp1; P.tmp2 = c->tmp2; P.tmp3 = c->tmp3; P.ctr = c->ctr;
    P.own_lo = 0; P.own_hi = 0x7fffffff;
    const unsigned grid = (unsigned)c->sm_count * 8u;
    k_scatter_edges_tris<<<dim3(grid, 2), 256, 0, c->stream>>>(P, ucap[1], ucap[2], c->k3_cap, ucap[3]);     // + the tets
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_CANONICAL + 1)) != AXB_OK) return st;
    if ((st = mark_event(c, AXB_ST_COUNT)) != AXB_OK) return st;
    {
        EmitAll E;
        E.n = (int)n; E.vkeep = c->vkeep; E.voff = c->voff; E.tmp1 = c->tmp1; E.tmp2 = c->tmp2; E.tmp3 = c->tmp3;
        E.off1 = c->off1; E.off2 = c->off2; E.off3 = c->off3; E.ctr = c->ctr;
        for (int d = 0; d < 4; ++d) { E.cap[d] = ucap[d]; E.out[d] = d_out[d]; }
        k_emit_all<<<dim3(grid, 4), 256, 0, c->stream>>>(E);
        LAUNCH_CHECK(c);
    }
    if ((st = mark_event(c, AXB_ST_COUNT + 1)) != AXB_OK) return st;
    k_publish_state<<<1, 32, 0, c->stream>>>(c->voff + n, c->off1 + n, c->off2 + n, c->off3 + n, c->ctr, c->h_dev->totals,
                                             &c->h_dev->ctr);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->state = S_PRUNED;                                    // the buckets were consumed
    if ((st = verify_assumed_edges(c)) != AXB_OK) return st;
    if (c->h->ctr.n_pq > c->pq_cap || c->h->ctr.n_pt > c->pt_cap || c->h->ctr.n_k3 > c->k3_cap)
        return AXB_ERR_ARENA + 1000;                       // a guessed list was too small: the caller redoes the stage
    if ((st = check_run_flags(c)) != AXB_OK) return st;
    c->n_pe = c->h->ctr.n_pe;
    c->n_pt = c->h->ctr.n_pt;
    c->n_pq = c->h->ctr.n_pq;
    for (int d = 0; d < 4; ++d) { c->counts[d] = c->h->totals[d]; counts[d] = c->counts[d]; }
    for (int d = 0; d < 4; ++d)
        if (c->counts[d] > (int64_t)ucap[d]) return AXB_ERR_ARENA + 1002;
    return AXB_OK;
}

}  // namespace

extern "C" int axb_potential(axb_ctx *c, int64_t lo, int64_t hi) {
    if (!c) return AXB_ERR_BAD_ARG;
    c->cull = false;          // the stage API exposes the complete potential levels
    return run_potential(c, lo, hi);
}

extern "C" int axb_potential_counts(const axb_ctx *c, int64_t counts[3]) {
    if (!c || !counts) return AXB_ERR_BAD_ARG;
    if (c->state < S_EDGES) return AXB_ERR_STATE;
    counts[0] = c->n_pe;
    counts[1] = c->state >= S_POTENTIAL ? c->n_pt : 0;
    counts[2] = c->state >= S_POTENTIAL ? c->n_pq : 0;
    return AXB_OK;
}

namespace {

// rows of one potential level as ascending ball indices + recomputed ortho data (generation order)
__global__ void k_export_potential(int what, unsigned m, const Atom *__restrict__ atoms, const int *__restrict__ orig,
                                   const int *__restrict__ pe_u, const int *__restrict__ pe_v,
                                   const int4 *__restrict__ pt, const int4 *__restrict__ pq_r, double eps_sing,
                                   int64_t *rows, double *centers, double *sizes) {
    unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int r[4] = {-1, -1, -1, -1};
    int k;
    if (what == AXB_PE) { r[0] = pe_u[e]; r[1] = pe_v[e]; k = 2; }
    else if (what == AXB_PT) { int4 q = pt[e]; r[0] = q.x; r[1] = q.y; r[2] = q.z; k = 3; }
    else { int4 q = pq_r[e]; r[0] = q.x; r[1] = q.y; r[2] = q.z; r[3] = q.w; k = 4; }
    Atom a[4];
    int o[4];
    for (int i = 0; i < k; ++i) { a[i] = load_atom(atoms, r[i]); o[i] = orig[r[i]]; }
    Ortho res;
    if (k == 2) res = ortho_edge(o[0], a[0], o[1], a[1], eps_sing);
    else if (k == 3) res = ortho_tri(o[0], a[0], o[1], a[1], o[2], a[2], eps_sing);
    else res = ortho_tet(o[0], a[0], o[1], a[1], o[2], a[2], o[3], a[3], eps_sing);
    for (int x = 1; x < k; ++x)
        for (int y = x; y > 0 && o[y - 1] > o[y]; --y) { int t = o[y]; o[y] = o[y - 1]; o[y - 1] = t; }
    if (rows) for (int i = 0; i < k; ++i) rows[(size_t)e * k + i] = o[i];
    if (centers) { centers[3 * (size_t)e] = res.cx; centers[3 * (size_t)e + 1] = res.cy; centers[3 * (size_t)e + 2] = res.cz; }
    if (sizes) sizes[e] = res.size;
}

}  // namespace

extern "C" int axb_potential_export(axb_ctx *c, int what, int64_t *d_rows, double *d_centers, double *d_sizes) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (what < AXB_PE || what > AXB_PQ) return fail(c, AXB_ERR_BAD_ARG, "what must be AXB_PE, AXB_PT or AXB_PQ");
    if (c->state < (what == AXB_PE ? S_EDGES : S_POTENTIAL)) return fail(c, AXB_ERR_STATE, "axb_potential_export: that level is not resident");
    if (what == AXB_PQ && c->pq_r == nullptr)
        return fail(c, AXB_ERR_STATE, "the potential-tet list is not materialised by axb_compute (fused path); use axb_potential");
    unsigned m = what == AXB_PE ? c->n_pe : (what == AXB_PT ? c->n_pt : c->n_pq);
    if (m) {
        k_export_potential<<<blocks_for(m, 128), 128, 0, c->stream>>>(what, m, c->atoms, c->orig, c->pe_u, c->pe_v, c->pt,
                                                                      c->pq_r, c->tol.eps_sing, d_rows, d_centers, d_sizes);
        LAUNCH_CHECK(c);
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return AXB_OK;
}

// ---- stage operations on resident or caller-supplied levels (stages.cuh) ----

extern "C" int axb_potential_edges(axb_ctx *c, int64_t lo, int64_t hi) {
    if (!c) return AXB_ERR_BAD_ARG;
    c->cull = false;
    return run_edges(c, lo, hi);
}

namespace {
// the triangle / tet counters back to their state after the edge stage (a stage may be run again)
int reset_simplex_counters(axb_ctx *c) {
    c->h->ctr.n_pt = 0; c->h->ctr.n_pq = 0; c->h->ctr.overflow = 0; c->h->ctr.tile_next = 0;
    c->h->ctr.err_key = ~0ull; c->h->ctr.err_count = 0;
    CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
    return AXB_OK;
}
}  // namespace

extern "C" int axb_potential_simplices(axb_ctx *c) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (c->state < S_EDGES) return fail(c, AXB_ERR_STATE, "axb_potential_simplices needs the potential edges first");
    c->cull = false;
    c->state = S_EDGES;
    int st = reset_simplex_counters(c);
    if (st != AXB_OK) return st;
    if ((st = mark_event(c, AXB_ST_POT_TRIANGLES)) != AXB_OK) return st;
    return run_tri_tet_lists(c);
}

extern "C" int axb_potential_import_edges(axb_ctx *c, const int64_t *d_rows, int64_t m) {
    if (!c || m < 0 || (m > 0 && !d_rows)) return AXB_ERR_BAD_ARG;
    if (c->state < S_GRID) return fail(c, AXB_ERR_STATE, "axb_potential_import_edges before axb_grid_build");
    if (c->slab_mode) return fail(c, AXB_ERR_STATE, "levels cannot be imported into a slab");
    if (m > 0xfffffff0ll) return fail(c, AXB_ERR_DENSITY, "more than 2^32 potential edges");
    const int n = (int)c->n;
    c->state = S_GRID;
    c->arena_used = c->mark_after_grid;
    c->rank_lo = 0; c->rank_hi = n; c->gen_lo = 0;
    c->dup_pending = false;
    memset(&c->h->ctr, 0, sizeof(Counters));
    c->h->ctr.err_key = ~0ull;
    c->h->ctr.first_bad = 0xffffffffu;
    c->h->ctr.n_pe = (unsigned)m;
    CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
    int st;
    if ((st = mark_event(c, AXB_ST_POT_EDGES)) != AXB_OK) return st;
    ARENA(c, c->adj_off, uint32_t, (size_t)n + 2);
    ARENA(c, c->deg, int, (size_t)n + 2);
    c->pe_cap = (uint32_t)std::max<int64_t>(m, 1);
    ARENA(c, c->pe_v, int, c->pe_cap);
    ARENA(c, c->pe_u, int, c->pe_cap);
    const size_t mark = c->arena_used;
    int *cursor;
    ARENA(c, cursor, int, (size_t)n + 2);
    CUDA_TRY(c, cudaMemsetAsync(c->deg, 0, sizeof(int) * ((size_t)n + 2), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(cursor, 0, sizeof(int) * ((size_t)n + 2), c->stream));
    if (m) {
        k_import_edge_count<<<blocks_for((size_t)m, 256), 256, 0, c->stream>>>(d_rows, (unsigned)m, n, c->rank, c->deg, c->ctr);
        LAUNCH_CHECK(c);
    }
    if ((st = device_scan(c, reinterpret_cast<const uint32_t *>(c->deg), (size_t)n, c->adj_off)) != AXB_OK) return st;
    if (m) {
        k_import_edge_scatter<<<blocks_for((size_t)m, 256), 256, 0, c->stream>>>(d_rows, (unsigned)m, n, c->rank, c->adj_off, cursor, c->pe_u, c->pe_v);
        LAUNCH_CHECK(c);
    }
    k_import_edge_order<<<blocks_for((size_t)n, 256), 256, 0, c->stream>>>(n, c->adj_off, c->deg, c->pe_v, c->ctr);
    LAUNCH_CHECK(c);
    if ((st = fetch_counters(c)) != AXB_OK) return st;
    c->arena_used = mark;
    if ((st = mark_event(c, AXB_ST_POT_EDGES + 1)) != AXB_OK) return st;
    if (c->h->ctr.overflow & (1u << 6)) return fail(c, AXB_ERR_BAD_ARG, "edge rows must hold two different ball indices in [0, n)");
    if (c->h->ctr.overflow & (1u << 7)) return fail(c, AXB_ERR_BAD_ARG, "edge rows hold the same edge twice");
    if (c->h->ctr.max_deg > (unsigned)AXB_MAX_PARTNERS)
        return fail(c, AXB_ERR_DENSITY, "a ball has more than %d potential-edge partners", AXB_MAX_PARTNERS);
    c->n_pe = (uint32_t)m;
    c->W = trimask_words(c->h->ctr.max_deg);
    if ((st = alloc_heavy(c)) != AXB_OK) return st;
    c->mark_after_edges = c->arena_used;
    c->state = S_EDGES;
    return AXB_OK;
}

namespace {
// allocate the triangle / tet lists after the edges and translate triangle rows into them
int import_triangles(axb_ctx *c, const int64_t *d_tri, int64_t m_t, uint32_t pq_cap) {
    c->arena_used = c->mark_after_edges;
    c->pt_cap = (uint32_t)std::max<int64_t>(m_t, 1);
    c->pq_cap = std::max<uint32_t>(pq_cap, 1);
    ARENA(c, c->pt, int4, c->pt_cap);
    ARENA(c, c->pq_r, int4, c->pq_cap);
    ARENA(c, c->pq_l, int, c->pq_cap);
    if (m_t) {
        k_import_simplices<<<blocks_for((size_t)m_t, 256), 256, 0, c->stream>>>(3, d_tri, (unsigned)m_t, (int)c->n, c->rank, c->adj_off,
                                                                             c->deg, c->pe_v, c->pt, c->pq_r, c->pq_l, c->ctr);
        LAUNCH_CHECK(c);
    }
    return AXB_OK;
}

int finish_import(axb_ctx *c) {
    int st = fetch_counters(c);
    if (st != AXB_OK) return st;
    if (c->h->ctr.overflow & (1u << 6))
        return fail(c, AXB_ERR_BAD_ARG, "a row names a ball outside [0, n), repeats one, or has an edge that is not in the edge level");
    if (c->h->ctr.err_key != ~0ull) return report_degenerate(c);
    c->n_pt = c->h->ctr.n_pt;
    c->n_pq = c->h->ctr.n_pq;
    c->k3_cap = c->pq_cap;
    c->many_tets = false;
    c->lists_complete = true;
    c->state = S_POTENTIAL;
    return AXB_OK;
}
}  // namespace

extern "C" int axb_potential_import_simplices(axb_ctx *c, const int64_t *d_tri, int64_t m_t, const int64_t *d_tet, int64_t m_q) {
    if (!c || m_t < 0 || m_q < 0 || (m_t > 0 && !d_tri) || (m_q > 0 && !d_tet)) return AXB_ERR_BAD_ARG;
    if (c->state < S_EDGES) return fail(c, AXB_ERR_STATE, "axb_potential_import_simplices needs the potential edges first");
    if (m_t > 0xfffffff0ll || m_q > 0xfffffff0ll) return fail(c, AXB_ERR_DENSITY, "more than 2^32 potential triangles or tetrahedra");
    c->state = S_EDGES;
    c->h->ctr.n_pt = (unsigned)m_t; c->h->ctr.n_pq = (unsigned)m_q; c->h->ctr.overflow = 0;
    c->h->ctr.err_key = ~0ull; c->h->ctr.err_count = 0;
    CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
    int st = import_triangles(c, d_tri, m_t, (uint32_t)m_q);
    if (st != AXB_OK) return st;
    if (m_q) {
        k_import_simplices<<<blocks_for((size_t)m_q, 256), 256, 0, c->stream>>>(4, d_tet, (unsigned)m_q, (int)c->n, c->rank, c->adj_off,
                                                                             c->deg, c->pe_v, c->pt, c->pq_r, c->pq_l, c->ctr);
        LAUNCH_CHECK(c);
    }
    return finish_import(c);
}

extern "C" int axb_potential_tets_from_triangles(axb_ctx *c, const int64_t *d_tri, int64_t m_t) {
    if (!c || m_t < 0 || (m_t > 0 && !d_tri)) return AXB_ERR_BAD_ARG;
    if (c->state < S_EDGES) return fail(c, AXB_ERR_STATE, "axb_potential_tets_from_triangles needs the potential edges first");
    if (m_t > 0xfffffff0ll) return fail(c, AXB_ERR_DENSITY, "more than 2^32 potential triangles");
    c->state = S_EDGES;
    uint64_t want = (uint64_t)m_t + 4096;
    for (int attempt = 0;; ++attempt) {
        if (want > 0xfffffff0ull) return fail(c, AXB_ERR_DENSITY, "more than 2^32 potential tetrahedra");
        c->h->ctr.n_pt = (unsigned)m_t; c->h->ctr.n_pq = 0; c->h->ctr.overflow = 0;
        c->h->ctr.err_key = ~0ull; c->h->ctr.err_count = 0;
        CUDA_TRY(c, cudaMemcpyAsync(c->ctr, &c->h->ctr, sizeof(Counters), cudaMemcpyHostToDevice, c->stream));
        int st = import_triangles(c, d_tri, m_t, (uint32_t)want);
        if (st != AXB_OK) return st;
        if (m_t) {
            TetsFromTris P;
            P.g = c->g; P.atoms = c->atoms; P.orig = c->orig; P.rank = c->rank; P.cell_of_rank = c->cell_of_rank;
            P.adj_off = c->adj_off; P.deg = c->deg; P.pe_v = c->pe_v; P.rows = d_tri; P.m = (unsigned)m_t;
            P.lim_a = c->tol.lim_a; P.eps_sing = c->tol.eps_sing;
            P.pq_r = c->pq_r; P.pq_l = c->pq_l; P.pq_cap = c->pq_cap; P.ctr = c->ctr; P.errs = c->errs; P.report_key = 0;
            k_tets_from_triangles<<<blocks_for((size_t)m_t, 128), 128, 0, c->stream>>>(P);
            LAUNCH_CHECK(c);
        }
        if ((st = fetch_counters(c)) != AXB_OK) return st;
        if (c->h->ctr.err_key != ~0ull && c->h->ctr.err_count > (unsigned)ERR_CAP) {
            // more singular solves than record slots: once more with only the first one (smallest key) reporting
            TetsFromTris P;
            P.g = c->g; P.atoms = c->atoms; P.orig = c->orig; P.rank = c->rank; P.cell_of_rank = c->cell_of_rank;
            P.adj_off = c->adj_off; P.deg = c->deg; P.pe_v = c->pe_v; P.rows = d_tri; P.m = (unsigned)m_t;
            P.lim_a = c->tol.lim_a; P.eps_sing = c->tol.eps_sing;
            P.pq_r = c->pq_r; P.pq_l = c->pq_l; P.pq_cap = 0; P.ctr = c->ctr; P.errs = c->errs; P.report_key = c->h->ctr.err_key;
            k_tets_from_triangles<<<blocks_for((size_t)m_t, 128), 128, 0, c->stream>>>(P);
            LAUNCH_CHECK(c);
            CUDA_TRY(c, cudaStreamSynchronize(c->stream));
            c->h->ctr.err_count = 1;
            return report_degenerate(c);
        }
        if (c->h->ctr.n_pq <= c->pq_cap) break;
        if (attempt >= 2) return fail(c, AXB_ERR_INTERNAL, "potential-tet buffer still too small after resize");
        want = (uint64_t)c->h->ctr.n_pq + 1024;
    }
    return finish_import(c);
}

extern "C" int axb_ac2_mask(axb_ctx *c, int what, uint8_t *d_mask) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (what < AXB_PE || what > AXB_PQ) return fail(c, AXB_ERR_BAD_ARG, "what must be AXB_PE, AXB_PT or AXB_PQ");
    if (c->state < (what == AXB_PE ? S_EDGES : S_POTENTIAL)) return fail(c, AXB_ERR_STATE, "axb_ac2_mask: that level is not resident");
    const unsigned m = what == AXB_PE ? c->n_pe : (what == AXB_PT ? c->n_pt : c->n_pq);
    if (m) {
        if (!d_mask) return AXB_ERR_BAD_ARG;
        k_ac2_mask<<<blocks_for(m, 128), 128, 0, c->stream>>>(what - AXB_PE, m, c->g, c->tol, c->atoms, c->orig, c->pe_u, c->pe_v, c->pt,
                                                              c->pq_r, d_mask);
        LAUNCH_CHECK(c);
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return AXB_OK;
}

// ---- alpha sweep with re-use (sweep.cuh) ----

extern "C" int axb_sweep_prepare(axb_ctx *c) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (c->state < S_POTENTIAL || !c->lists_complete || c->slab_mode || c->rank_lo != 0 || c->rank_hi != (int)c->n)
        return fail(c, AXB_ERR_STATE, "axb_sweep_prepare needs the complete potential levels of the whole input (axb_potential(0, n))");
    c->state = S_POTENTIAL;
    c->sweep_on = false;
    c->sweep_ready = false;
    c->sweep_ranked = false;
    const unsigned E = c->n_pe, T = c->n_pt, Q = c->n_pq;
    // the lists end at pt_cap / pq_cap; everything the sweep keeps across alphas sits behind them
    ARENA(c, c->sw.esize, double, std::max(E, 1u));
    ARENA(c, c->sw.pf, unsigned char, std::max(E, 1u));
    ARENA(c, c->sw.ac2e, unsigned char, std::max(E, 1u));
    ARENA(c, c->sw.tsize, double, std::max(T, 1u));
    ARENA(c, c->sw.tvw, int, std::max(T, 1u));
    ARENA(c, c->sw.ac2t, unsigned char, std::max(T, 1u));
    ARENA(c, c->sw.qsize, double, std::max(Q, 1u));
    ARENA(c, c->sw.qtsize, double, std::max(Q, 1u));
    ARENA(c, c->sw.qe, int4, std::max(Q, 1u));
    ARENA(c, c->sw.ac2q, unsigned char, std::max(Q, 1u));
    c->mark_after_sweep = c->arena_used;
    CUDA_TRY(c, cudaMemsetAsync(&c->ctr->n_k3, 0, sizeof(unsigned int) * PRUNE_COUNTER_WORDS, c->stream));
    PruneParams P = prune_params(c);
    if (E) { k_sweep_prepare_edges<<<blocks_for(E, SWEEP_THREADS), SWEEP_THREADS, 0, c->stream>>>(P, E, c->sw); LAUNCH_CHECK(c); }
    if (T) { k_sweep_prepare_tris<<<blocks_for(T, SWEEP_THREADS), SWEEP_THREADS, 0, c->stream>>>(P, T, c->sw); LAUNCH_CHECK(c); }
    if (Q) { k_sweep_prepare_tets<<<blocks_for(Q, SWEEP_THREADS), SWEEP_THREADS, 0, c->stream>>>(P, Q, c->sw); LAUNCH_CHECK(c); }
    int st = fetch_counters(c);
    if (st != AXB_OK) return st;
    if ((st = check_run_flags(c)) != AXB_OK) return st;
    c->sweep_ready = true;
    return AXB_OK;
}

extern "C" int axb_sweep_prune(axb_ctx *c, double alpha) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (!c->sweep_ready || c->state < S_POTENTIAL) return fail(c, AXB_ERR_STATE, "axb_sweep_prune before axb_sweep_prepare");
    if (!(alpha <= c->prm.alpha)) return fail(c, AXB_ERR_BAD_ARG, "the sweep was prepared for alpha <= %.17g", c->prm.alpha);
    if (c->prm.biomolecule && alpha < 0.0) return fail(c, AXB_ERR_BAD_ARG, "biomolecule mode requires alpha >= 0");
    c->state = S_POTENTIAL;
    c->arena_used = c->mark_after_sweep;
    c->tol.lim_a = alpha + c->prm.eps_abs;
    for (int i = AXB_ST_PRUNE_TETS; i < AXB_ST_COUNT + 2; ++i) c->ev_set[i] = false;
    int st = mark_event(c, AXB_ST_PRUNE_TETS);
    if (st != AXB_OK) return st;
    if (c->n_pe) {
        k_sweep_edge_flags<<<blocks_for(c->n_pe, 256), 256, 0, c->stream>>>(c->n_pe, c->atoms, c->pe_u, c->pe_v, c->sw.esize, alpha,
                                                                            c->prm.eps_abs, c->sw.pf);
        LAUNCH_CHECK(c);
    }
    c->sweep_on = true;
    st = run_prune(c);
    c->sweep_on = false;
    return st;
}

extern "C" int axb_sweep_rank(axb_ctx *c, const double *alphas, int k) {
    if (!c || !alphas || k < 1 || k > 254) return AXB_ERR_BAD_ARG;
    if (!c->sweep_ready || c->state < S_POTENTIAL) return fail(c, AXB_ERR_STATE, "axb_sweep_rank before axb_sweep_prepare");
    for (int q = 0; q < k; ++q) {
        if (!(alphas[q] <= c->prm.alpha) || (q && !(alphas[q - 1] < alphas[q])))
            return fail(c, AXB_ERR_BAD_ARG, "alphas must ascend strictly and stay <= %.17g, the alpha the sweep was prepared for", c->prm.alpha);
        if (c->prm.biomolecule && alphas[q] < 0.0) return fail(c, AXB_ERR_BAD_ARG, "biomolecule mode requires alpha >= 0");
    }
    c->state = S_POTENTIAL;
    c->sweep_ranked = false;
    c->arena_used = c->mark_after_sweep;
    const unsigned E = c->n_pe, T = c->n_pt, Q = c->n_pq;
    const size_t n = (size_t)c->n;
    SweepArrays &S = c->sw;
    double *d_alphas;
    ARENA(c, d_alphas, double, (size_t)k);
    ARENA(c, S.ke, unsigned char, std::max(E, 1u));
    ARENA(c, S.ae, unsigned, std::max(E, 1u));
    ARENA(c, S.at, unsigned, std::max(T, 1u));
    ARENA(c, S.aq, unsigned, std::max(Q, 1u));
    const size_t ones_from = c->arena_used;                   // "never" / "no triangle yet": all bits set
    ARENA(c, S.av, unsigned, n + 1);
    ARENA(c, S.row_first, unsigned, std::max(E, 1u));
    const size_t ones_to = c->arena_used;
    ARENA(c, S.ptmask, unsigned long long, (size_t)std::max(E, 1u) * c->W);
    S.alphas = d_alphas;
    S.K = k;
    CUDA_TRY(c, cudaMemcpyAsync(d_alphas, alphas, sizeof(double) * (size_t)k, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->arena + ones_from, 0xff, ones_to - ones_from, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(S.ptmask, 0, sizeof(unsigned long long) * (size_t)std::max(E, 1u) * c->W, c->stream));
    PruneParams P = prune_params(c);
    if (E) { k_sweep_rank_edges<<<blocks_for(E, 256), 256, 0, c->stream>>>(P, E, S); LAUNCH_CHECK(c); }
    if (T) {
        k_sweep_tri_index<<<blocks_for(T, 256), 256, 0, c->stream>>>(P, T, S); LAUNCH_CHECK(c);
        k_sweep_rank_tris<<<blocks_for(T, 256), 256, 0, c->stream>>>(P, T, S); LAUNCH_CHECK(c);
    }
    if (Q) { k_sweep_rank_tets<<<blocks_for(Q, 256), 256, 0, c->stream>>>(P, Q, S); LAUNCH_CHECK(c); }
    if (T) { k_sweep_inherit_tris<<<blocks_for(T, 256), 256, 0, c->stream>>>(P, T, S); LAUNCH_CHECK(c); }
    if (E) { k_sweep_inherit_edges<<<blocks_for(E, 256), 256, 0, c->stream>>>(P, E, S); LAUNCH_CHECK(c); }
    k_sweep_rank_vertices<<<blocks_for(n, 256), 256, 0, c->stream>>>(P, S);
    LAUNCH_CHECK(c);
    int st = fetch_counters(c);
    if (st != AXB_OK) return st;
    if (c->h->ctr.overflow & (1u << 8))
        return fail(c, AXB_ERR_STATE, "a face of a listed tetrahedron is not a listed triangle (rounding): use axb_sweep_prune for this input");
    c->mark_after_sweep = c->arena_used;                      // the ranks stay; every alpha's kept state comes behind them
    c->sweep_ranked = true;
    return AXB_OK;
}

extern "C" int axb_sweep_select(axb_ctx *c, int index) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (!c->sweep_ranked || c->state < S_POTENTIAL) return fail(c, AXB_ERR_STATE, "axb_sweep_select before axb_sweep_rank");
    if (index < 0 || index >= c->sw.K) return fail(c, AXB_ERR_BAD_ARG, "alpha index out of range");
    c->state = S_POTENTIAL;
    c->arena_used = c->mark_after_sweep;
    for (int i = AXB_ST_PRUNE_TETS; i < AXB_ST_COUNT + 2; ++i) c->ev_set[i] = false;
    int st = mark_event(c, AXB_ST_PRUNE_TETS);
    if (st != AXB_OK) return st;
    if ((st = alloc_prune_arrays(c, false)) != AXB_OK) return st;
    PruneParams P = prune_params(c);
    k_sweep_select<<<(unsigned)c->sm_count * 8u, 256, 0, c->stream>>>(P, c->sw, (unsigned)index, c->n_pe, c->n_pt, c->n_pq);
    LAUNCH_CHECK(c);
    for (int i = AXB_ST_PRUNE_TETS + 1; i <= AXB_ST_PRUNE_VERTICES + 1; ++i)
        if ((st = mark_event(c, i)) != AXB_OK) return st;
    c->state = S_PRUNED;
    return AXB_OK;
}

extern "C" int axb_prune(axb_ctx *c) {
    if (!c) return AXB_ERR_BAD_ARG;
    return run_prune(c);
}

extern "C" int axb_canonicalize(axb_ctx *c, int64_t counts[4]) {
    if (!c) return AXB_ERR_BAD_ARG;
    int st = run_canonicalize(c, counts);
    if (st == AXB_ERR_ARENA + 1000) return fail(c, AXB_ERR_INTERNAL, "potential buffers overflowed; call axb_potential again");
    return st;
}

extern "C" int axb_export(axb_ctx *c, int64_t *d_v, int64_t *d_e, int64_t *d_t, int64_t *d_q) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (c->state < S_CANON) return fail(c, AXB_ERR_STATE, "axb_export before axb_canonicalize");
    int st;
    if ((st = mark_event(c, AXB_ST_COUNT)) != AXB_OK) return st;
    if (d_v) {
        k_emit_vertices<int64_t><<<blocks_for((size_t)c->n, 256), 256, 0, c->stream>>>((int)c->n, c->vkeep, c->voff, c->gidx, d_v, 0xffffffffu);
        LAUNCH_CHECK(c);
    }
    if (d_e && c->counts[1]) {
        k_emit_edges<PlainOut<int64_t>><<<blocks_for((size_t)c->counts[1], 256), 256, 0, c->stream>>>(c->tmp1, c->off1, (unsigned)c->counts[1], nullptr, c->gidx, PlainOut<int64_t>{d_e}, c->ctr);
        LAUNCH_CHECK(c);
    }
    if (d_t && c->counts[2]) {
        k_emit_tris<PlainOut<int64_t>><<<blocks_for((size_t)c->counts[2], 256), 256, 0, c->stream>>>(c->tmp2, c->off2, (unsigned)c->counts[2], nullptr, c->gidx, PlainOut<int64_t>{d_t}, c->ctr);
        LAUNCH_CHECK(c);
    }
    if (d_q && c->counts[3]) {
        k_emit_tets<PlainOut<int64_t>><<<blocks_for((size_t)c->counts[3], 256), 256, 0, c->stream>>>(c->tmp3, c->off3, (unsigned)c->counts[3], nullptr, c->gidx, PlainOut<int64_t>{d_q}, c->ctr);
        LAUNCH_CHECK(c);
    }
    return mark_event(c, AXB_ST_COUNT + 1);
}

extern "C" int axb_sync_check(axb_ctx *c) {
    if (!c) return AXB_ERR_BAD_ARG;
    int st = fetch_counters(c);
    if (st != AXB_OK) return st;
    return check_run_flags(c);
}

namespace {
// grid -> potential levels (optimistic list sizes, cull mode) -> pruning kernels, all queued; returns after the edge
// stage's sync, with about two thirds of the step's GPU work still in flight
int compute_start(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *prm) {
    c->defer_dup = true;
    int st = axb_grid_build(c, n, d_xyz, d_radii, prm);
    c->defer_dup = false;
    if (st != AXB_OK) return st;
    c->cull = true;
    if (const char *e = getenv("AXB_CULL")) c->cull_mask = atoi(e);
    c->allow_assume = true;
    st = run_potential(c, 0, n, /*optimistic=*/true);
    c->allow_assume = false;
    if (st == AXB_OK) st = run_prune(c);
    if (st != AXB_OK) c->cull = false;
    return st;
}

// canonical lists (bucketed for axb_export, or straight into caller buffers); redoes the triangle / tet stage with exact
// sizes if a guessed list size did not hold
int compute_finish(axb_ctx *c, int64_t counts[4], int64_t *const d_out[4], const int64_t cap[4]) {
    auto canon = [&]() { return d_out ? run_canonicalize_into(c, counts, d_out, cap) : run_canonicalize(c, counts); };
    int st = canon();
    if (st == AXB_ERR_ARENA + 1001) {                       // the remembered edge-stage sizes did not hold: once more, waiting for them
        c->memo.valid = false;
        c->edges_assumed = false;
        st = run_potential(c, 0, c->n, /*optimistic=*/true);
        if (st == AXB_OK) st = run_prune(c);
        if (st == AXB_OK) st = canon();
    }
    if (st == AXB_ERR_ARENA + 1000) {
        st = run_tri_tet_lists(c, false, /*redo=*/true);
        if (st == AXB_OK) st = run_prune(c);
        if (st == AXB_OK) st = canon();
        if (st == AXB_ERR_ARENA + 1000) st = fail(c, AXB_ERR_INTERNAL, "a potential list overflowed after it was sized exactly");
    }
    if (st == AXB_OK || st == AXB_ERR_ARENA + 1002) remember_edges(c);
    else c->memo.valid = false;
    if (st == AXB_ERR_ARENA + 1002)
        st = fail(c, AXB_ERR_STATE, "a result list is longer than the caller's buffer (%lld %lld %lld %lld rows); use axb_compute + axb_export",
                  (long long)counts[0], (long long)counts[1], (long long)counts[2], (long long)counts[3]);
    c->cull = false;
    return st;
}
}  // namespace

extern "C" int axb_compute(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *prm,
                           int64_t counts[4]) {
    if (!c) return AXB_ERR_BAD_ARG;
    int st = compute_start(c, n, d_xyz, d_radii, prm);
    return st != AXB_OK ? st : compute_finish(c, counts, nullptr, nullptr);
}

extern "C" int axb_compute_start(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *prm) {
    if (!c) return AXB_ERR_BAD_ARG;
    return compute_start(c, n, d_xyz, d_radii, prm);
}

extern "C" int axb_compute_finish_into(axb_ctx *c, int64_t *d_v, int64_t *d_e, int64_t *d_t, int64_t *d_q,
                                       const int64_t capacity[4], int64_t counts[4]) {
    if (!c || !capacity || !counts || !d_v || !d_e || !d_t || !d_q) return AXB_ERR_BAD_ARG;
    if (c->state != S_PRUNED || !c->cull) return fail(c, AXB_ERR_STATE, "axb_compute_finish_into needs axb_compute_start first");
    int64_t *const out[4] = {d_v, d_e, d_t, d_q};
    return compute_finish(c, counts, out, capacity);
}

extern "C" int axb_compute_into(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii, const axb_params *prm,
                                int64_t *d_v, int64_t *d_e, int64_t *d_t, int64_t *d_q, const int64_t capacity[4],
                                int64_t counts[4]) {
    if (!c) return AXB_ERR_BAD_ARG;
    int st = compute_start(c, n, d_xyz, d_radii, prm);
    return st != AXB_OK ? st : axb_compute_finish_into(c, d_v, d_e, d_t, d_q, capacity, counts);
}

extern "C" int axb_compute_slab(axb_ctx *c, int64_t n, const double *d_xyz, const double *d_radii,
                                const int64_t *d_global_index, const axb_params *prm, const axb_slab *slab,
                                int64_t z_own_lo, int64_t z_own_hi, int64_t counts[4]) {
    if (!c || !slab) return AXB_ERR_BAD_ARG;
    int st = axb_grid_build_slab(c, n, d_xyz, d_radii, d_global_index, prm, slab);
    if (st != AXB_OK) return st;
    int64_t lo = 0, hi = 0;
    if ((st = axb_slab_rank_range(c, z_own_lo, z_own_hi, &lo, &hi)) != AXB_OK) return st;
    c->cull = true;
    st = run_potential(c, lo, hi);
    c->cull = false;
    if (st != AXB_OK) return st;
    if ((st = run_prune(c)) != AXB_OK) return st;
    st = run_canonicalize(c, counts);
    if (st == AXB_ERR_ARENA + 1000) return fail(c, AXB_ERR_INTERNAL, "a potential list overflowed after it was sized exactly");
    return st;
}

namespace {

int ensure_pool(axb_ctx *c) {
    if (c->pool) return AXB_OK;
    unsigned hw = std::thread::hardware_concurrency();
    // the calling thread helps too; two cores stay free for the CUDA driver's own threads (measured:
    // 14 of 16 beats 16 of 16, which gets preempted in the middle of tasks)
    unsigned workers = std::max(3u, std::min(32u, hw ? hw : 4u)) - 3u;
    if (const char *e = getenv("AXB_WIDEN_THREADS")) workers = (unsigned)std::max(0, atoi(e) - 1);
    c->pool = new (std::nothrow) axb::WidenPool(workers);
    if (!c->pool) return fail(c, AXB_ERR_INTERNAL, "cannot create the host worker threads");
    return AXB_OK;
}

// below this many bytes a job's host-side marshalling (input staging, row widening) runs on the calling thread
constexpr size_t SMALL_JOB_BYTES = (size_t)1 << 20;

bool is_pinned(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type != cudaMemoryTypeUnregistered;
}

// Inputs to the device.  Pinned buffers go straight to the copy engine.  Pageable ones (a plain numpy array)
// would make the driver stage them through its own bounce buffer on ONE thread (~10 GB/s: 3 ms per million
// balls); instead the host threads copy them into a pinned staging area in 8 MiB slices and each slice is handed to
// the copy engine as soon as it is complete, so the DMA of one slice overlaps the memcpy of the next.
int upload_inputs(axb_ctx *c, int64_t n, const double *h_xyz, const double *h_radii, double *d_in) {
    const size_t bx = (size_t)n * 3 * sizeof(double), br = (size_t)n * sizeof(double);
    // small inputs (one protein): the driver's own bounce buffer is faster than waking the staging threads
    if (bx + br <= SMALL_JOB_BYTES || (is_pinned(h_xyz) && is_pinned(h_radii))) {
        CUDA_TRY(c, cudaMemcpyAsync(d_in, h_xyz, bx, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(d_in + 3 * (size_t)n, h_radii, br, cudaMemcpyHostToDevice, c->stream));
        return AXB_OK;
    }
    int st = ensure_pool(c);
    if (st != AXB_OK) return st;
    if (c->h_in_bytes < bx + br) {
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));      // a previous upload may still read the old area
        if (c->h_in) cudaFreeHost(c->h_in);
        c->h_in = nullptr;
        c->h_in_bytes = 0;
        const size_t want = (bx + br) + (bx + br) / 4;
        CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void **>(&c->h_in), want, cudaHostAllocDefault));
        c->h_in_bytes = want;
    } else {
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));      // the area is reused: the previous run's DMA must be over
    }
    timespec ts0;
    clock_gettime(CLOCK_MONOTONIC, &ts0);
    const size_t slice = getenv("AXB_UPLOAD_SLICE") ? (size_t)atol(getenv("AXB_UPLOAD_SLICE")) : ((size_t)8 << 20);
    const char *src[2] = {reinterpret_cast<const char *>(h_xyz), reinterpret_cast<const char *>(h_radii)};
    const size_t len[2] = {bx, br};
    size_t off = 0;
    for (int part = 0; part < 2; ++part) {
        for (size_t lo = 0; lo < len[part]; lo += slice) {
            const size_t m = std::min(slice, len[part] - lo);
            c->pool->begin(m / ((size_t)256 << 10) + 4);
            c->pool->publish_copy(src[part] + lo, c->h_in + off + lo, m, (size_t)256 << 10);
            c->pool->finish();
            CUDA_TRY(c, cudaMemcpyAsync(reinterpret_cast<char *>(d_in) + off + lo, c->h_in + off + lo, m, cudaMemcpyHostToDevice, c->stream));
        }
        off += len[part];
    }
    if (getenv("AXB_TRACE")) {
        timespec ts1;
        clock_gettime(CLOCK_MONOTONIC, &ts1);
        fprintf(stderr, "[axb] staged upload of %zu bytes queued after %.3f ms\n", bx + br,
                (ts1.tv_sec - ts0.tv_sec) * 1e3 + (ts1.tv_nsec - ts0.tv_nsec) * 1e-6);
    }
    return AXB_OK;
}

}  // namespace

extern "C" int axb_compute_host(axb_ctx *c, int64_t n, const double *h_xyz, const double *h_radii, const axb_params *prm,
                                int64_t counts[4]) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (n <= 0) return fail(c, AXB_ERR_EMPTY, "at least one ball is required");
    if (!h_xyz || !h_radii) return fail(c, AXB_ERR_BAD_ARG, "null input pointer");
    // inputs live at the END of the arena so the per-run bump allocator never touches them
    size_t in_bytes = ((size_t)n * 4 * sizeof(double) + ARENA_ALIGN - 1) / ARENA_ALIGN * ARENA_ALIGN;
    if (!c->arena || c->arena_bytes < in_bytes + ARENA_ALIGN) {
        c->arena_needed = in_bytes + axb_arena_hint(n, prm ? prm->alpha : 0.0, 1.9);
        return fail(c, AXB_ERR_ARENA, "scratch arena too small for the input copy");
    }
    double *d_in = reinterpret_cast<double *>(c->arena + c->arena_bytes - in_bytes);
    CUDA_TRY(c, cudaSetDevice(c->device));
    {
        int up = upload_inputs(c, n, h_xyz, h_radii, d_in);
        if (up != AXB_OK) return up;
    }
    const size_t full = c->arena_bytes;
    c->arena_bytes = full - in_bytes;
    int st = axb_compute(c, n, d_in, d_in + 3 * (size_t)n, prm, counts);
    c->arena_bytes = full;
    if (st == AXB_ERR_ARENA) c->arena_needed += in_bytes;
    return st;
}

// ---- pipelined host path: the D2H copy of a finished dimension overlaps the remaining kernels ----
// begin: inputs up, grid, potential stage; returns row CAPACITIES for the four host arrays (tight upper
// bounds: K0 <= n, K1 <= potential edges, K2 <= ~potential triangles, K3 <= potential tets).
// finish: tets are final after their prune kernel -> canonicalise + start their copy on a second stream;
// then triangles, edges, vertices the same way; one synchronisation at the very end.
extern "C" int axb_compute_host_begin(axb_ctx *c, int64_t n, const double *h_xyz, const double *h_radii,
                                      const axb_params *prm, int64_t capacity[4]) {
    if (!c || !capacity) return AXB_ERR_BAD_ARG;
    if (n <= 0) return fail(c, AXB_ERR_EMPTY, "at least one ball is required");
    if (!h_xyz || !h_radii) return fail(c, AXB_ERR_BAD_ARG, "null input pointer");
    size_t in_bytes = ((size_t)n * 4 * sizeof(double) + ARENA_ALIGN - 1) / ARENA_ALIGN * ARENA_ALIGN;
    if (!c->arena || c->arena_bytes < in_bytes + ARENA_ALIGN) {
        c->arena_needed = in_bytes + axb_arena_hint(n, prm ? prm->alpha : 0.0, 1.9);
        return fail(c, AXB_ERR_ARENA, "scratch arena too small for the input copy");
    }
    double *d_in = reinterpret_cast<double *>(c->arena + c->arena_bytes - in_bytes);
    CUDA_TRY(c, cudaSetDevice(c->device));
    {
        int up = upload_inputs(c, n, h_xyz, h_radii, d_in);
        if (up != AXB_OK) return up;
    }
    const size_t full = c->arena_bytes;
    c->arena_bytes = full - in_bytes;
    auto now_ms = []() { timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e3 + t.tv_nsec * 1e-6; };
    const double tb0 = now_ms();
    c->defer_dup = true;
    int st = axb_grid_build(c, n, d_in, d_in + 3 * (size_t)n, prm);
    c->defer_dup = false;
    const double tb1 = now_ms();
    if (st == AXB_OK) {
        c->cull = true;
        st = run_potential(c, 0, n);
        c->cull = false;
    }
    if (getenv("AXB_TRACE")) fprintf(stderr, "[axb] begin: grid (incl. upload wait) %.3f ms, potential %.3f ms\n", tb1 - tb0, now_ms() - tb1);
    c->arena_bytes = full;
    if (st == AXB_ERR_ARENA) c->arena_needed += in_bytes;
    if (st != AXB_OK) return st;
    capacity[0] = n;
    capacity[1] = c->n_pe;
    capacity[2] = (int64_t)c->n_pt + c->n_pt / 8 + 1024;     // inherited faces outside the potential list are rare
    capacity[3] = c->n_pq;
    for (int d = 0; d < 4; ++d) c->host_cap[d] = capacity[d];
    return AXB_OK;
}

#ifndef AXB_WIRE_DEFAULT
#define AXB_WIRE_DEFAULT 0
#endif

namespace {
// A row count goes to the host as a zero-copy store from a one-thread kernel, NOT as a 4-byte
// cudaMemcpyAsync: that would queue on the same D2H copy engine behind megabytes of row chunks and
// stall the compute stream until they have drained.
__global__ void k_publish_total(const uint32_t *__restrict__ src, uint32_t *host_dst) {
    *host_dst = *src;
    __threadfence_system();
}

size_t D2H_CHUNK = (size_t)1 << 19;                // int32 elements per D2H copy (2 MiB; AXB_D2H_CHUNK overrides)
constexpr size_t WIDEN_PIECE = (size_t)1 << 16;    // int32 elements per widening task

struct PoolRun {                                   // every exit path closes the pool run
    axb::WidenPool *pool;
    ~PoolRun() { if (pool) pool->finish(); }
};
struct PendingChunk { cudaEvent_t ev; const int32_t *src; int64_t *dst; size_t n; int dim; size_t row0; };
}  // namespace

extern "C" int axb_compute_host_finish(axb_ctx *c, int64_t *h_v, int64_t *h_e, int64_t *h_t, int64_t *h_q,
                                       int64_t counts[4]) {
    if (!c || !counts) return AXB_ERR_BAD_ARG;
    if (c->state != S_POTENTIAL) return fail(c, AXB_ERR_STATE, "axb_compute_host_finish needs axb_compute_host_begin first");
    const size_t n = (size_t)c->n;
    int st = alloc_prune_arrays(c, false);
    if (st != AXB_OK) return st;
    int64_t *h[4] = {h_v, h_e, h_t, h_q};
    // What crosses PCIe per row: int32 values, widened by the host threads; nothing at all for the vertices
    // when every vertex is kept.  Optional compact formats (AXB_WIRE bit 0: edges send only their second
    // column, bit 1: triangles their last two; the owner column is rebuilt on the host from the per-owner row
    // offsets, which travel once) cut the PCIe bytes by another third, but on the 16-core host measured here
    // the row expansion then becomes the bottleneck (finish 2.9 ms instead of 2.4 ms at 1M atoms), so they
    // are off by default.
    const int wire_mode = getenv("AXB_WIRE") ? atoi(getenv("AXB_WIRE")) : AXB_WIRE_DEFAULT;
    const bool compact1 = (wire_mode & 1) != 0, compact2 = (wire_mode & 2) != 0;
    const int wire_width[4] = {1, compact1 ? 1 : 2, compact2 ? 2 : 3, 4};
    // 24-bit wire (default while every ball index fits): edges, triangles and tets cross PCIe as three bytes per
    // value -- per D2H chunk a plane of low halves and a plane of high bytes (canon.cuh: Packed24Out) -- and the
    // host threads unpack them straight into the int64 rows.  AXB_WIRE24=0 switches it off.
    const bool p24 = wire_mode == 0 && n < ((size_t)1 << 24) && !(getenv("AXB_WIRE24") && atoi(getenv("AXB_WIRE24")) == 0);
    if (const char *e = getenv("AXB_D2H_CHUNK")) D2H_CHUNK = std::max<size_t>(1 << 14, (size_t)atol(e));
    size_t rows_per_chunk_of[4];
    unsigned rows_shift[4];
    for (int d = 0; d < 4; ++d) {
        rows_per_chunk_of[d] = std::max<size_t>(1, D2H_CHUNK / (size_t)wire_width[d]);
        rows_shift[d] = 1;                                    // 24-bit planes: a power of two of whole rows per chunk
        while (((size_t)2 << rows_shift[d]) <= rows_per_chunk_of[d]) ++rows_shift[d];
        if (p24 && d >= 1) rows_per_chunk_of[d] = (size_t)1 << rows_shift[d];
    }
    int32_t *d_out[4];
    size_t stage_off[4], stage_elems = 0;
    for (int d = 0; d < 4; ++d) {
        const size_t elems = (size_t)std::max<int64_t>(c->host_cap[d], 1) * wire_width[d];
        ARENA(c, d_out[d], int32_t, elems);
        stage_off[d] = stage_elems;
        stage_elems += (elems + 63) / 64 * 64;
    }
    size_t stage_offsets[3] = {0, 0, 0};              // staged copies of off1 / off2 (index = dimension)
    for (int d = 1; d <= 2; ++d) {
        stage_offsets[d] = stage_elems;
        stage_elems += (n + 2 + 63) / 64 * 64;
    }
    ARENA(c, c->off1, uint32_t, n + 2);
    ARENA(c, c->off2, uint32_t, n + 2);
    ARENA(c, c->off3, uint32_t, n + 2);
    ARENA(c, c->voff, uint32_t, n + 2);
    ARENA(c, c->tmp1, int2, (size_t)std::max<int64_t>(c->host_cap[1], 1));
    ARENA(c, c->tmp2, int4, (size_t)std::max<int64_t>(c->host_cap[2], 1));
    ARENA(c, c->tmp3, int4, (size_t)std::max<int64_t>(c->host_cap[3], 1));
    // pinned staging area + widening threads (created once, grown on demand)
    if (c->h_stage_elems < stage_elems) {
        if (c->h_stage) cudaFreeHost(c->h_stage);
        c->h_stage = nullptr;
        c->h_stage_elems = 0;
        const size_t want = stage_elems + stage_elems / 4;
        CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void **>(&c->h_stage), want * sizeof(int32_t), cudaHostAllocDefault));
        c->h_stage_elems = want;
    }
    if ((st = ensure_pool(c)) != AXB_OK) return st;
    // one event per D2H chunk: a chunk holds rows_per_chunk_of[d] whole rows, which can be fewer values than D2H_CHUNK
    // (24-bit planes round the rows down to a power of two), so count chunks per dimension
    size_t max_chunks = 8;
    for (int d = 0; d < 4; ++d)
        max_chunks += ((size_t)std::max<int64_t>(c->host_cap[d], 1) + rows_per_chunk_of[d] - 1) / rows_per_chunk_of[d] + 1;
    auto grow_events = [&](size_t want) -> int {
        while (c->chunk_ev.size() < want) {
            cudaEvent_t e;
            CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->chunk_ev.push_back(e);
        }
        return AXB_OK;
    };
    if ((st = grow_events(max_chunks)) != AXB_OK) return st;
    PruneParams P = prune_params(c);
    CanonParams Q;
    Q.n = (int)n; Q.orig = c->orig; Q.adj_off = c->adj_off; Q.pe_u = c->pe_u; Q.pe_v = c->pe_v; Q.pe_cap = c->pe_cap;
    Q.W = c->W; Q.trimask = c->trimask; Q.eflag = c->eflag; Q.k3 = c->k3;
    Q.cnt1 = c->cnt1; Q.cnt2 = c->cnt2; Q.cnt3 = c->cnt3; Q.off1 = c->off1; Q.off2 = c->off2; Q.off3 = c->off3;
    Q.tmp1 = c->tmp1; Q.tmp2 = c->tmp2; Q.tmp3 = c->tmp3; Q.ctr = c->ctr;
    Q.own_lo = 0; Q.own_hi = 0x7fffffff;
    const unsigned grid = (unsigned)c->sm_count * 8u;
    // Everything is queued up front.  After the scan of a dimension its exact row count goes to the
    // host (4 bytes + an event); the host follows those events, queues the copies of exactly the valid
    // rows on the second stream in 2 MiB chunks (behind the event that marks the rows complete) and
    // hands every chunk that has landed to the widening threads.
    auto mark_total = [&](int d, const uint32_t *off_end) -> int {
        k_publish_total<<<1, 1, 0, c->stream>>>(off_end, &c->h_dev->totals[d]);
        LAUNCH_CHECK(c);
        CUDA_TRY(c, cudaEventRecord(c->dim_count[d], c->stream));
        return AXB_OK;
    };
    auto mark_ready = [&](int d) -> int {
        CUDA_TRY(c, cudaEventRecord(c->dim_ready[d], c->stream));
        return AXB_OK;
    };
    // tets
    // few tets per thread: static grid-stride; many (large alpha, dense cores): dynamic 64-tet claims
    if ((uint64_t)c->n_pq > (uint64_t)c->n + c->n / 2)
        k_prune_tets<1><<<(unsigned)c->sm_count * (unsigned)TETS_MINB, 256, 0, c->stream>>>(P);
    else
        k_prune_tets<0><<<(unsigned)c->sm_count * (unsigned)TETS_GRID, 256, 0, c->stream>>>(P);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_TETS + 1)) != AXB_OK) return st;
    if ((st = device_scan(c, c->cnt3, n, c->off3)) != AXB_OK) return st;
    if ((st = mark_total(3, c->off3 + n)) != AXB_OK) return st;
    k_scatter_tets<<<grid, 256, 0, c->stream>>>(Q, c->k3_cap, (unsigned)std::min<int64_t>(c->host_cap[3], 0xfffffff0ll));
    LAUNCH_CHECK(c);
    if (p24) k_emit_tets<Packed24Out><<<grid, 256, 0, c->stream>>>(c->tmp3, c->off3, (unsigned)c->host_cap[3], c->off3 + n, nullptr, Packed24Out{reinterpret_cast<unsigned char *>(d_out[3]), rows_shift[3]}, c->ctr);
    else k_emit_tets<PlainOut<int32_t>><<<grid, 256, 0, c->stream>>>(c->tmp3, c->off3, (unsigned)c->host_cap[3], c->off3 + n, nullptr, PlainOut<int32_t>{d_out[3]}, c->ctr);
    LAUNCH_CHECK(c);
    if ((st = mark_ready(3)) != AXB_OK) return st;
    // triangles
    k_prune_tris<<<(unsigned)c->sm_count * (unsigned)PRUNE_GRID, TRIS_THREADS, 0, c->stream>>>(P);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_TRIANGLES + 1)) != AXB_OK) return st;
    if ((st = device_scan(c, c->cnt2, n, c->off2)) != AXB_OK) return st;
    if ((st = mark_total(2, c->off2 + n)) != AXB_OK) return st;
    k_scatter_tris<<<grid, 256, 0, c->stream>>>(Q, (unsigned)c->host_cap[2]);
    LAUNCH_CHECK(c);
    if (p24) k_emit_tris<Packed24Out, false><<<grid, 256, 0, c->stream>>>(c->tmp2, c->off2, (unsigned)c->host_cap[2], c->off2 + n, nullptr, Packed24Out{reinterpret_cast<unsigned char *>(d_out[2]), rows_shift[2]}, c->ctr);
    else if (compact2) k_emit_tris<PlainOut<int32_t>, true><<<grid, 256, 0, c->stream>>>(c->tmp2, c->off2, (unsigned)c->host_cap[2], c->off2 + n, nullptr, PlainOut<int32_t>{d_out[2]}, c->ctr);
    else k_emit_tris<PlainOut<int32_t>, false><<<grid, 256, 0, c->stream>>>(c->tmp2, c->off2, (unsigned)c->host_cap[2], c->off2 + n, nullptr, PlainOut<int32_t>{d_out[2]}, c->ctr);
    LAUNCH_CHECK(c);
    if ((st = mark_ready(2)) != AXB_OK) return st;
    // edges
    k_prune_edges<<<(unsigned)c->sm_count * (unsigned)PRUNE_GRID, PRUNE_THREADS, 0, c->stream>>>(P);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_EDGES + 1)) != AXB_OK) return st;
    if ((st = device_scan(c, c->cnt1, n, c->off1)) != AXB_OK) return st;
    if ((st = mark_total(1, c->off1 + n)) != AXB_OK) return st;
    k_scatter_edges<<<grid, 256, 0, c->stream>>>(Q, (unsigned)c->host_cap[1]);
    LAUNCH_CHECK(c);
    if (p24) k_emit_edges<Packed24Out, false><<<grid, 256, 0, c->stream>>>(c->tmp1, c->off1, (unsigned)c->host_cap[1], c->off1 + n, nullptr, Packed24Out{reinterpret_cast<unsigned char *>(d_out[1]), rows_shift[1]}, c->ctr);
    else if (compact1) k_emit_edges<PlainOut<int32_t>, true><<<grid, 256, 0, c->stream>>>(c->tmp1, c->off1, (unsigned)c->host_cap[1], c->off1 + n, nullptr, PlainOut<int32_t>{d_out[1]}, c->ctr);
    else k_emit_edges<PlainOut<int32_t>, false><<<grid, 256, 0, c->stream>>>(c->tmp1, c->off1, (unsigned)c->host_cap[1], c->off1 + n, nullptr, PlainOut<int32_t>{d_out[1]}, c->ctr);
    LAUNCH_CHECK(c);
    if ((st = mark_ready(1)) != AXB_OK) return st;
    // vertices
    k_prune_vertices<<<blocks_for(n, 256), 256, 0, c->stream>>>(P, c->rank_lo, c->rank_hi);
    LAUNCH_CHECK(c);
    if ((st = mark_event(c, AXB_ST_PRUNE_VERTICES + 1)) != AXB_OK) return st;
    if ((st = device_scan(c, c->vkeep, n, c->voff)) != AXB_OK) return st;
    if ((st = mark_total(0, c->voff + n)) != AXB_OK) return st;
    k_emit_vertices<int32_t><<<blocks_for(n, 256), 256, 0, c->stream>>>((int)n, c->vkeep, c->voff, nullptr, d_out[0], 0xffffffffu);
    LAUNCH_CHECK(c);
    if ((st = mark_ready(0)) != AXB_OK) return st;
    if ((st = mark_event(c, AXB_ST_CANONICAL + 1)) != AXB_OK) return st;

    // the host follows the GPU dimension by dimension, feeds the copy stream and the widening threads
    static const bool trace = getenv("AXB_TRACE") != nullptr;
    auto now_ms = []() { timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e3 + t.tv_nsec * 1e-6; };
    const double t_q = now_ms();
    double t_dim[4] = {0, 0, 0, 0};
    c->pool->begin(2 * (stage_elems / WIDEN_PIECE) + 2 * max_chunks + n / WIDEN_PIECE + 16,
                   /*inline_run=*/stage_elems * sizeof(int32_t) <= SMALL_JOB_BYTES);
    PoolRun run{c->pool};
    std::vector<PendingChunk> chunks;
    chunks.reserve(max_chunks);
    size_t pumped = 0;
    c->last_d2h_bytes = 0;
    auto pump = [&](bool block) -> int {              // publish every chunk that has landed, in order
        while (pumped < chunks.size()) {
            const PendingChunk &k = chunks[pumped];
            cudaError_t e = block ? cudaEventSynchronize(k.ev) : cudaEventQuery(k.ev);
            if (e == cudaErrorNotReady) return AXB_OK;
            if (e != cudaSuccess) return fail(c, AXB_ERR_CUDA, "D2H chunk failed: %s", cudaGetErrorString(e));
            if (k.dim == 1 && compact1)
                c->pool->publish(axb::WK_EDGE_ROWS, k.src, k.dst, k.n, WIDEN_PIECE, 1, 2,
                                 reinterpret_cast<const uint32_t *>(c->h_stage + stage_offsets[1]), n, k.row0);
            else if (k.dim == 2 && compact2)
                c->pool->publish(axb::WK_TRI_ROWS, k.src, k.dst, k.n, WIDEN_PIECE / 2, 2, 3,
                                 reinterpret_cast<const uint32_t *>(c->h_stage + stage_offsets[2]), n, k.row0);
            else if (k.dim >= 1 && p24)
                c->pool->publish(axb::WK_UNPACK24, k.src, k.dst, k.n, WIDEN_PIECE, 0, 1, nullptr, k.n, 0);
            else
                c->pool->publish(axb::WK_WIDEN, k.src, k.dst, k.n, WIDEN_PIECE, 1, 1, nullptr, 0, 0);
            ++pumped;
        }
        return AXB_OK;
    };
    for (int d = 3; d >= 0; --d) {
        for (;;) {
            cudaError_t e = cudaEventQuery(c->dim_count[d]);
            if (e == cudaSuccess) break;
            if (e != cudaErrorNotReady) return fail(c, AXB_ERR_CUDA, "row count of dimension %d: %s", d, cudaGetErrorString(e));
            if ((st = pump(false)) != AXB_OK) return st;
        }
        c->counts[d] = c->h->totals[d];
        t_dim[d] = now_ms();
        if (c->counts[d] > c->host_cap[d]) {
            cudaStreamSynchronize(c->stream);
            cudaStreamSynchronize(c->copy_stream);
            return fail(c, AXB_ERR_STATE, "dimension %d has %lld rows, more than the %lld the capacity bound allowed; use axb_compute_host + axb_export_host",
                        d, (long long)c->counts[d], (long long)c->host_cap[d]);
        }
        if (h[d] && c->counts[d]) {
            if (d == 0 && c->counts[0] == (int64_t)n) {       // every vertex kept: 0, 1, ..., n - 1
                c->pool->publish(axb::WK_IOTA, nullptr, h[0], n, WIDEN_PIECE, 0, 1, nullptr, 0, 0);
                continue;
            }
            const size_t rows = (size_t)c->counts[d];
            const size_t w = (size_t)wire_width[d];
            const size_t rows_per_chunk = rows_per_chunk_of[d];
            int32_t *stage = c->h_stage + stage_off[d];
            if (d >= 1 && p24) {                              // 3 bytes per value; chunk q starts 3 * q * chunk_vals bytes in
                CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->dim_ready[d], 0));
                const char *dev = reinterpret_cast<const char *>(d_out[d]);
                char *hst = reinterpret_cast<char *>(stage);
                for (size_t lo = 0; lo < rows; lo += rows_per_chunk) {
                    const size_t m = std::min(rows_per_chunk, rows - lo);
                    if ((st = grow_events(chunks.size() + 1)) != AXB_OK) return st;
                    cudaEvent_t ev = c->chunk_ev[chunks.size()];
                    CUDA_TRY(c, cudaMemcpyAsync(hst + lo * w * 3, dev + lo * w * 3, m * w * 3, cudaMemcpyDeviceToHost, c->copy_stream));
                    CUDA_TRY(c, cudaEventRecord(ev, c->copy_stream));
                    chunks.push_back(PendingChunk{ev, reinterpret_cast<const int32_t *>(hst + lo * w * 3), h[d] + lo * w, m * w, d, 0});
                }
                c->last_d2h_bytes += (int64_t)(rows * w * 3);
                continue;
            }
            const bool compact = (d == 1 && compact1) || (d == 2 && compact2);
            if (compact) {                                    // the row offsets per owner were final before the count was
                const uint32_t *off = d == 1 ? c->off1 : c->off2;
                CUDA_TRY(c, cudaMemcpyAsync(c->h_stage + stage_offsets[d], off, (n + 1) * sizeof(uint32_t),
                                            cudaMemcpyDeviceToHost, c->copy_stream));
                c->last_d2h_bytes += (int64_t)((n + 1) * sizeof(uint32_t));
            }
            CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->dim_ready[d], 0));
            for (size_t lo = 0; lo < rows; lo += rows_per_chunk) {
                const size_t m = std::min(rows_per_chunk, rows - lo);
                if ((st = grow_events(chunks.size() + 1)) != AXB_OK) return st;
                cudaEvent_t ev = c->chunk_ev[chunks.size()];
                CUDA_TRY(c, cudaMemcpyAsync(stage + lo * w, d_out[d] + lo * w, m * w * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                            c->copy_stream));
                CUDA_TRY(c, cudaEventRecord(ev, c->copy_stream));
                // plain dimensions are widened value by value, edges / triangles row by row
                if (compact) chunks.push_back(PendingChunk{ev, stage + lo * w, h[d] + lo * (d + 1), m, d, lo});
                else chunks.push_back(PendingChunk{ev, stage + lo * w, h[d] + lo * w, m * w, d, 0});
            }
            c->last_d2h_bytes += (int64_t)(rows * w * sizeof(int32_t));
        }
    }
    if ((st = pump(true)) != AXB_OK) return st;
    const double t_landed = now_ms();
    run.pool = nullptr;
    c->pool->finish();
    if (trace)
        fprintf(stderr, "[axb] finish: counts known at +%.3f %.3f %.3f %.3f ms (tets..vertices), last chunk landed +%.3f, widened +%.3f (%zu chunks)\n",
                t_dim[3] - t_q, t_dim[2] - t_q, t_dim[1] - t_q, t_dim[0] - t_q, t_landed - t_q, now_ms() - t_q, chunks.size());
    if ((st = fetch_counters(c)) != AXB_OK) return st;
    CUDA_TRY(c, cudaStreamSynchronize(c->copy_stream));
    if ((st = check_run_flags(c)) != AXB_OK) return st;
    for (int d = 0; d < 4; ++d) counts[d] = c->counts[d];
    c->state = S_PRUNED;      // the buckets were consumed; axb_export is not available after this path
    return AXB_OK;
}

extern "C" int64_t axb_last_d2h_bytes(const axb_ctx *c) { return c ? c->last_d2h_bytes : 0; }

extern "C" int axb_export_host(axb_ctx *c, int64_t *h_v, int64_t *h_e, int64_t *h_t, int64_t *h_q) {
    if (!c) return AXB_ERR_BAD_ARG;
    if (c->state < S_CANON) return fail(c, AXB_ERR_STATE, "axb_export_host before axb_canonicalize");
    const size_t mark = c->arena_used;
    int64_t *d[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t *h[4] = {h_v, h_e, h_t, h_q};
    for (int k = 0; k < 4; ++k)
        if (h[k]) ARENA(c, d[k], int64_t, (size_t)std::max<int64_t>(c->counts[k], 1) * (k + 1));
    int st = axb_export(c, d[0], d[1], d[2], d[3]);
    if (st != AXB_OK) return st;
    for (int k = 0; k < 4; ++k)
        if (h[k] && c->counts[k])
            CUDA_TRY(c, cudaMemcpyAsync(h[k], d[k], sizeof(int64_t) * (size_t)c->counts[k] * (k + 1), cudaMemcpyDeviceToHost, c->stream));
    st = axb_sync_check(c);
    c->arena_used = mark;
    return st;
}

// -------------------------------------------------------------------- merge

extern "C" int axb_merge_rows(axb_ctx *c, int k, int64_t n_index, const int64_t *d_rows, int64_t m, int64_t *d_out,
                              int64_t *count_out) {
    return axb_merge_rows_range(c, k, 0, n_index, d_rows, m, d_out, count_out);
}

extern "C" int axb_merge_rows_range(axb_ctx *c, int k, int64_t index_lo, int64_t index_hi, const int64_t *d_rows, int64_t m,
                                    int64_t *d_out, int64_t *count_out) {
    const int64_t n_index = index_hi - index_lo, base = index_lo;
    if (!c || k < 1 || k > 4 || index_lo < 0 || n_index < 1 || m < 0 || !count_out) return AXB_ERR_BAD_ARG;
    if (n_index >= ((int64_t)1 << 31) - 1 || m >= ((int64_t)1 << 32) - 16) return fail(c, AXB_ERR_BAD_ARG, "merge input too large");
    c->state = S_NONE;          // the arena is reused from the start
    c->arena_used = 0;
    c->arena_needed = 0;
    *count_out = 0;
    if (m == 0) return AXB_OK;
    if (!d_rows || !d_out) return fail(c, AXB_ERR_BAD_ARG, "null pointer");
    CUDA_TRY(c, cudaSetDevice(c->device));
    uint32_t *cnt, *off, *ucnt, *uoff;
    int4 *tmp;
    unsigned char *dup;
    ARENA(c, c->ctr, Counters, 1);
    ARENA(c, cnt, uint32_t, (size_t)n_index + 2);
    ARENA(c, off, uint32_t, (size_t)n_index + 2);
    ARENA(c, ucnt, uint32_t, (size_t)n_index + 2);
    ARENA(c, uoff, uint32_t, (size_t)n_index + 2);
    ARENA(c, tmp, int4, (size_t)m);
    ARENA(c, dup, unsigned char, (size_t)m);
    CUDA_TRY(c, cudaMemsetAsync(c->ctr, 0, sizeof(Counters), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * ((size_t)n_index + 2), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(ucnt, 0, sizeof(uint32_t) * ((size_t)n_index + 2), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(tmp, 0xff, sizeof(int4) * (size_t)m, c->stream));   // owner -1 = skipped
    const unsigned nb = blocks_for((size_t)m, 256);
    k_merge_count<<<nb, 256, 0, c->stream>>>(d_rows, (unsigned)m, k, (unsigned)n_index, base, cnt, c->ctr);
    LAUNCH_CHECK(c);
    int st = device_scan(c, cnt, (size_t)n_index, off);
    if (st != AXB_OK) return st;
    k_merge_scatter<<<nb, 256, 0, c->stream>>>(d_rows, (unsigned)m, k, (unsigned)n_index, base, cnt, off, tmp);
    LAUNCH_CHECK(c);
    k_merge_mark<<<nb, 256, 0, c->stream>>>(tmp, off, (unsigned)m, ucnt, dup);
    LAUNCH_CHECK(c);
    st = device_scan(c, ucnt, (size_t)n_index, uoff);
    if (st != AXB_OK) return st;
    k_merge_emit<<<nb, 256, 0, c->stream>>>(tmp, off, uoff, dup, (unsigned)m, k, base, d_out);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaMemcpyAsync(&c->h->totals[0], uoff + n_index, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    st = fetch_counters(c);
    if (st != AXB_OK) return st;
    if (c->h->ctr.overflow) return fail(c, AXB_ERR_BAD_ARG, "merge input holds a first index outside the given range");
    *count_out = c->h->totals[0];
    return AXB_OK;
}

// ------------------------------------------------------------------- probes

namespace {
__global__ void k_ortho_batch(int64_t m, int k, const double *__restrict__ pts, const double *__restrict__ r2,
                              double eps_sing, double *centers, double *sizes, uint8_t *singular) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    Atom a[4];
    for (int i = 0; i < k; ++i) {
        a[i].x = pts[(s * k + i) * 3]; a[i].y = pts[(s * k + i) * 3 + 1]; a[i].z = pts[(s * k + i) * 3 + 2];
        a[i].r2 = r2[s * k + i];
    }
    Ortho o;
    if (k == 1) { o.cx = a[0].x; o.cy = a[0].y; o.cz = a[0].z; o.size = -a[0].r2; o.singular = false; }
    else if (k == 2) o = ortho2(a[0], a[1], eps_sing);
    else if (k == 3) { Atom p[3] = {a[0], a[1], a[2]}; o = orthoN<3>(p, eps_sing); }
    else { Atom p[4] = {a[0], a[1], a[2], a[3]}; o = orthoN<4>(p, eps_sing); }
    centers[3 * s] = o.cx; centers[3 * s + 1] = o.cy; centers[3 * s + 2] = o.cz;
    sizes[s] = o.size;
    singular[s] = o.singular ? 1 : 0;
}
}  // namespace

extern "C" int axb_ortho_batch(axb_ctx *c, int64_t m, int k, const double *d_pts, const double *d_r2, double eps_sing,
                               double *d_centers, double *d_sizes, uint8_t *d_singular) {
    if (!c || k < 1 || k > 4 || m < 0) return AXB_ERR_BAD_ARG;
    if (m == 0) return AXB_OK;
    k_ortho_batch<<<blocks_for((size_t)m, 128), 128, 0, c->stream>>>(m, k, d_pts, d_r2, eps_sing, d_centers, d_sizes, d_singular);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return AXB_OK;
}


// ------------------------------------------------------------ canonical text
// write_complex (reference io.py:228-236): one line per simplex, "dim v0 [v1 [v2 [v3]]]\n", in
// (dimension, lexicographic) order -- which is the order of the four arrays.  Pure host code
// (threads over row ranges: sizes, prefix, write); no GPU involved.

namespace {

inline int dec_len(int64_t v) {
    int n = 1;
    uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
    while (u >= 10) { u /= 10; ++n; }
    return n + (v < 0 ? 1 : 0);
}

inline char *put_dec(char *p, int64_t v) {
    char tmp[24];
    int n = 0;
    uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
    do { tmp[n++] = (char)('0' + u % 10); u /= 10; } while (u);
    if (v < 0) *p++ = '-';
    while (n) *p++ = tmp[--n];
    return p;
}

struct RowSpan { int dim; int64_t lo, hi; const int64_t *rows; int64_t bytes; };

}  // namespace

extern "C" int axb_format_complex(const int64_t counts[4], const int64_t *v, const int64_t *e, const int64_t *t,
                                  const int64_t *q, char *out, int64_t capacity, int64_t *needed) {
    if (!counts || !needed) return AXB_ERR_BAD_ARG;
    const int64_t *arr[4] = {v, e, t, q};
    for (int d = 0; d < 4; ++d)
        if (counts[d] < 0 || (counts[d] > 0 && !arr[d])) return AXB_ERR_BAD_ARG;
    unsigned nthreads = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<RowSpan> spans;
    for (int d = 0; d < 4; ++d) {
        const int64_t chunk = std::max<int64_t>(1 << 16, (counts[d] + nthreads - 1) / nthreads);
        for (int64_t lo = 0; lo < counts[d]; lo += chunk)
            spans.push_back({d, lo, std::min(counts[d], lo + chunk), arr[d], 0});
    }
    auto for_spans = [&](auto fn) {
        std::vector<std::thread> pool;
        std::atomic<size_t> next{0};
        const unsigned workers = (unsigned)std::min<size_t>(nthreads, std::max<size_t>(1, spans.size()));
        for (unsigned w = 0; w < workers; ++w)
            pool.emplace_back([&]() { for (size_t i; (i = next.fetch_add(1)) < spans.size();) fn(spans[i]); });
        for (auto &th : pool) th.join();
    };
    for_spans([](RowSpan &s) {
        const int k = s.dim + 1;
        int64_t b = 0;
        for (int64_t r = s.lo; r < s.hi; ++r) {
            b += 2;                                          // dim digit + newline
            for (int c = 0; c < k; ++c) b += 1 + dec_len(s.rows[r * k + c]);   // space + number
        }
        s.bytes = b;
    });
    int64_t total = 0;
    std::vector<int64_t> offset(spans.size());
    for (size_t i = 0; i < spans.size(); ++i) { offset[i] = total; total += spans[i].bytes; }
    *needed = total;
    if (!out || capacity < total) return out ? AXB_ERR_ARENA : AXB_OK;
    std::vector<char *> where(spans.size());
    for (size_t i = 0; i < spans.size(); ++i) where[i] = out + offset[i];
    for_spans([&](RowSpan &s) {
        char *p = where[&s - spans.data()];
        const int k = s.dim + 1;
        for (int64_t r = s.lo; r < s.hi; ++r) {
            *p++ = (char)('0' + s.dim);
            for (int c = 0; c < k; ++c) { *p++ = ' '; p = put_dec(p, s.rows[r * k + c]); }
            *p++ = '\n';
        }
    });
    return AXB_OK;
}
