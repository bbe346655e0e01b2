// Level-0 -> level-1 Galerkin product without the assembled level-0 matrix (used with the
// matrix-free level-0 operator, matfree.cuh).
//
// PAPER.md Eq. 6 refreshes A_1 = P^T A_0 P every outer iteration.  With A_0 = H H^T +
// diag(at) (reading c14) and the aggregate-wise prolongator (k = 1, reading c6):
//   G_{a,v}  = sum_{i in a, v in verts(i)} P_i h_{i,v}                       (3-vector per (vertex, aggregate) pair)
//   (A_1)_ab = sum_v G_{a,v} . G_{b,v}  +  [a == b] sum_{i in a} P_i^2 at_i
// which is P^T A_0 P exactly (up to rounding order).  The pattern of A_1 is the one va_coarse_pattern
// (or galerkin_symbolic) built; a setup-time plan maps every (v, a, b) product to its coarse entry.
// Off-diagonal entries: one thread each; diagonal entries (10-50x the products): one warp each.
#pragma once
#include "common.cuh"

namespace mgpbd {

struct VaPlan {
    int64_t npairs = 0, ncontrib = 0, cnnz = 0, ninc = 0;
    int64_t hv_stride = 0;  // plane stride of the vertex-major copy hv (padded layout: npad)
    DBuf<int32_t> vlist2;   // incidence codes (constraint*kc + slot) per vertex sorted by (agg, code)
    DBuf<int32_t> vpos;     // ninc: position of vlist2[e] in the matrix-free hv planes (padded layout) or vlist
    DBuf<int32_t> pstart;   // npairs + 1: incidence range of (vertex, aggregate) pair p in vlist2
    DBuf<int64_t> cptr;     // cnnz + 1: products of coarse entry k
    DBuf<int2> cpq;         // ncontrib: (p, q) pair indices, grouped by coarse entry, ascending (v, p, q)
    DBuf<int2> crange;      // cnnz: product range of off-diagonal entry k in cpq; (0, 0) for diagonals
    DBuf<unsigned char> G;  // npairs x 4 values of the hot type
};

// Setup time: the coarse pattern of A_1 = P^T A_0 P from the mesh alone — (a, b) is an entry iff some
// vertex is touched by members of both aggregates (reading c14: A_ij != 0 iff constraints i, j share a
// vertex) — off-diagonals ascending, diagonal last; replaces galerkin_symbolic of level 0 when the
// hot loop is matrix-free.
void va_coarse_pattern(int32_t nv, int kc, const int64_t* vptr, const int32_t* vlist, const int32_t* agg,
                       int32_t n_agg, DBuf<int64_t>& crowptr, DBuf<int32_t>& ccol, cudaStream_t s);

// at_i = alpha_i / dt^2 (fp64, all rows) for the setup-time product
void va_at(int32_t m, const double* alpha, double dt, double* at, cudaStream_t s);

// Setup time, after aggregation and the coarse pattern of level 1.
// ppos / hv_stride: the matrix-free operator's padded vertex-major layout (matfree.cuh) that va_numeric's
// hv argument uses (nullptr: hv indexed like vlist).
void va_symbolic(int32_t nv, int kc, const int64_t* vptr, const int32_t* vlist, const int32_t* agg, int32_t n_agg,
                 const int64_t* crowptr, const int32_t* ccol, int64_t cnnz, VaPlan& plan, cudaStream_t s,
                 const int64_t* ppos = nullptr, int64_t hv_stride = 0);

// Every outer iteration: cval = A_1 values from the current h (m x kc x 3), P and at = alpha/dt^2 (all
// m rows); cdinv = 1/diag.  hv (optional, nullptr = read h): the matrix-free operator's vertex-major
// copy of h over ALL incidences (single-rank layout).  No allocation (graph-capturable).
template <class T>
void va_numeric(VaPlan& plan, int kc, const T* h, const T* hv, const T* P, const int64_t* mptr,
                const int32_t* mlist, const T* at, int32_t n_agg, const int64_t* crowptr, T* cval, T* cdinv,
                cudaStream_t s);

}  // namespace mgpbd
