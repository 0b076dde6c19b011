// common.cuh -- shared device-side types and warp helpers.
//
// Everything on the device lives in "rank space": atoms are stored in the
// order of the reference's Grid.order (grid.py:128, sorted by (cell key, ball
// index)), so a cell, a row of cells along x and therefore every (2r+1)^3
// neighbourhood row is a contiguous range of ranks.  Ball indices of the
// caller ("orig") only reappear when simplices are emitted.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace axb {

struct __align__(32) Atom {   // one 32-byte sector per atom
    double x, y, z, r2;
};

// Device view of the uniform grid (reference grid.py:30-39), dense cell table.
struct GridView {
    double ox, oy, oz;        // origin
    double side;              // cell side sqrt(r_max^2 + alpha)
    int dx, dy, dz;           // dims of the LOCAL table (dz = loaded z layers)
    int z_lo;                 // first loaded z layer of the global grid (0 unless this is a slab)
    int dz_glob;              // z layers of the global grid (== dz unless this is a slab)
    int n;                    // balls
    const uint32_t *cell_start;   // dense mode: (n_cells + 1) exclusive prefix of per-cell counts
    const long long *skeys;       // sparse mode (cell_start == nullptr): the n cell keys in rank order (ascending);
                                  // the reference's implicit storage (grid.py:38-39, 76-88) without the table
};

// Scalar run parameters needed by the predicate kernels.
struct Tol {
    double lim_a;             // alpha + eps_abs         (pipeline.py:358)
    double eps_abs;
    double eps_sing;
    double r2max;             // largest squared radius of the input (AC2 reach bound)
    double reach_max;         // upper bound of every ball's reach sqrt(r^2 + alpha + eps_abs) (edge candidate bound)
};

// Device-side counters / status block (one per context, zeroed per run).
struct Counters {
    unsigned long long err_key;        // min over (stage, generator rank, ordinal) of singular solves
    unsigned long long pair_bound;     // sum over generators of C(deg, 2)
    unsigned int n_pe;                 // potential edges
    unsigned int n_pt;                 // potential triangles
    unsigned int n_pq;                 // potential tets
    unsigned int max_deg;
    unsigned int err_count;            // singular records appended
    unsigned int dup_count;            // duplicate-centre records appended
    unsigned int overflow;             // bit0: partner cap, bit1: PT cap, bit2: PQ cap, bit3: lookup miss
    unsigned int first_bad;            // first non-finite ball index (0xffffffff = none)
    unsigned int tile_next;            // k_tri_tet3: next unclaimed tile (dynamic scheduling)
    unsigned int n_heavy;              // generators with more partners than a k_tri_tet3 tile holds (heavy.cuh)
    // --- the pruning stage's own counters: adjacent, zeroed with one memset per prune run
    unsigned int n_k3;                 // kept tets
    unsigned int lookup_miss;          // inherited faces whose generator row has no such partner
    unsigned int work_next[3];         // prune kernels (tets, triangles, edges): next unclaimed chunk
};
constexpr int PRUNE_COUNTER_WORDS = 5; // n_k3 .. work_next[2]

constexpr int ERR_CAP = 1024;          // singular records kept per run
constexpr int DUP_CAP = 4096;

struct ErrRecord {
    unsigned long long key;
    int verts[4];                      // ball indices ascending, -1 padded
    int nverts;
    int pad;
};

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, v, o);
        if (lane_id() >= o) v += t;
    }
    return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// error key: stage (3 bits) | generator rank (31 bits) | ordinal (29 bits); smaller = raised first
// by the reference when the whole input is one chunk (pipeline.py:357, 414, 419, 477).
enum { ST_EDGE = 1, ST_VW = 2, ST_TRI = 3, ST_TET = 4 };
constexpr int ERR_ORD_BITS = 29;
__device__ __forceinline__ unsigned long long make_err_key(int stage, int gen_rank, unsigned ordinal) {
    return ((unsigned long long)stage << 60) | ((unsigned long long)(unsigned)gen_rank << ERR_ORD_BITS) |
           (ordinal & ((1u << ERR_ORD_BITS) - 1u));
}

// partner slots of a tet inside its generator's list, three to a word (a generator has fewer than 1024 partners:
// AXB_MAX_PARTNERS)
constexpr int SLOT_BITS = 10;
constexpr int SLOT_MASK = (1 << SLOT_BITS) - 1;
__host__ __device__ __forceinline__ int pack_slots(int i, int j, int k) { return i | (j << SLOT_BITS) | (k << (2 * SLOT_BITS)); }
// ordinal of a tet in its generator's enumeration: (ordinal of the generating triangle, third partner slot)
__device__ __forceinline__ unsigned tet_ordinal(unsigned tri_ord, int k) { return (tri_ord << SLOT_BITS) | (unsigned)k; }

}  // namespace axb
