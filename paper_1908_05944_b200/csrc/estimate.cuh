// estimate.cuh -- shared parameter block and helpers of the estimation kernels
// (stage one of the reference, pipeline.py:316-479).
// Potential edges: edges.cuh.  Potential triangles and tets: estimate3.cuh.
#pragma once

#include "common.cuh"
#include "predicates.cuh"

namespace axb {

constexpr int MAXP = 1023;     // AXB_MAX_PARTNERS (partner slots are packed 10 bits each)

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
    int *pq_l;                  // potential tets, partner slots (pack_slots)
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

__device__ __forceinline__ int nth_set_bit(unsigned long long m, int n) {
    for (int q = 0; q < n; ++q) m &= m - 1;
    return __ffsll((long long)m) - 1;
}

}  // namespace axb
