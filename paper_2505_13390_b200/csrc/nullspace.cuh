// k > 1 near-kernel variant of the setup and solve ("We repeat this six
// times to generate six distinct B", "R of QR decomposition serves as B at the next level";
// readings c23-c25).
//
// Every level stays a scalar CSR matrix (each coarse DOF is a node of the next level's aggregation).
// Aggregate a of level l owns r_a <= k consecutive coarse DOFs coff[a] .. coff[a+1]-1; the prolongator is
// P = blockdiag_a(Q_a) with Q_a the thin-QR factor of the aggregate's k near-kernel columns.
//   * QR (qr_prolongator): warp per aggregate, modified Gram-Schmidt with one re-orthogonalisation pass,
//     columns in order; a column is dropped when its orthogonal remainder is <= rank_tol of its norm;
//     a zero block gets the uniform column.  Output: P as CSR (row i: r_agg(i) entries), the member-major
//     copy Qs (restriction), coff, the DOF -> aggregate map and B_next = R (n_next x k, column-major).
//   * Galerkin (kgal_*): the aggregate-level plan of the k = 1 product (galerkin_symbolic: segments of
//     fine entries grouped by (fine row, aggregate of the column)) drives a block product:
//       stage 1, per segment t = (i, b):   W_t[d] = sum_{e in t} A_e P_{col(e), d}          (d < r_b)
//       stage 2, per aggregate entry (a,b): (A_c)_{(a,c),(b,d)} = sum_{t in list(a,b)} P_{row(t), c} W_t[d]
//     written into the block-expanded coarse CSR (off-diagonals ascending, diagonal last).
#pragma once
#include "common.cuh"
#include "setup.cuh"

namespace mgpbd {

struct KProlongator {
    int k = 1;
    int32_t n = 0, n_agg = 0, nc = 0;
    DBuf<int32_t> coff;      // n_agg + 1
    DBuf<int32_t> dof_agg;   // nc: aggregate of each coarse DOF
    DBuf<double> Qs64;       // n x k, member slot major (mptr order): Qs[(slot)*k + j]
    DBuf<int64_t> pptr;      // n + 1
    DBuf<int32_t> pcol;      // pptr[n]
    DBuf<double> pval64;     // pptr[n]
};

// QR injection of the k columns of B (column-major n x k) over the aggregates (mptr/mlist ascending).
// Returns n_next (= coff[n_agg]); B_next receives R (n_next x k, column-major).  Host-synchronising.
int32_t qr_prolongator(int32_t n, int32_t n_agg, int k, const int32_t* agg, const int64_t* mptr,
                       const int32_t* mlist, const double* B, double rank_tol, KProlongator& P,
                       DBuf<double>& B_next, cudaStream_t s);

// Block-expanded coarse pattern from the aggregate-level pattern (arow/acol: off-diagonals ascending,
// diagonal last) and the DOF offsets: xrow/xcol (nc + 1 / nnz) and, per aggregate-level entry, the
// offset of its block inside the expanded rows (xoff, counted in ascending column order) and its
// aggregate row (erow).
void kgal_expand(int32_t n_agg, const int64_t* arow, const int32_t* acol, const int32_t* coff, DBuf<int64_t>& xrow,
                 DBuf<int32_t>& xcol, DBuf<int64_t>& xoff, DBuf<int32_t>& erow, cudaStream_t s);

// Numeric block Galerkin of one level: fine CSR (rowptr/col/val), plan (aggregate level), P (pptr, pval in
// T), aggregate pattern (arow/acol, xoff), expanded pattern (xrow) -> cval / cdinv (nullptr: skip).
// W: plan.T * k scratch.
template <class T>
void kgal_numeric(const GalerkinPlan& plan, const int64_t* rowptr, const int32_t* col, const T* val, int k,
                  const int64_t* pptr, const T* pval, const int32_t* coff, const int32_t* agg, int32_t n_agg,
                  const int32_t* erow, const int32_t* acol, const int64_t* xoff, const int64_t* xrow, int32_t nc,
                  T* W, T* cval, T* cdinv, cudaStream_t s);

// V-cycle transfer with the general prolongator: b_c = P^T r (DOF-major over the aggregate's members,
// ascending, fixed order) and x += P e (row-major over P's row).
template <class T>
void krestrict(int32_t nc, int k, const int32_t* dof_agg, const int32_t* coff, const int64_t* mptr,
               const int32_t* mlist, const T* Qs, const T* r, T* bc, cudaStream_t s);
template <class T>
void kprolong(int32_t row0, int32_t rows, const int64_t* pptr, const int32_t* pcol, const T* pval, const T* e, T* x,
              cudaStream_t s);

}  // namespace mgpbd
