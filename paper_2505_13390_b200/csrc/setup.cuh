// AMG setup kernels and the Galerkin product (a7).
// Setup always runs on fp64 values; the numeric Galerkin product is templated on the hot precision.
#pragma once
#include <functional>

#include "common.cuh"
#include "solve.cuh"

namespace mgpbd {

// Filter: strong[e] = (col != i) && |A_ij| >= theta sqrt(|A_ii||A_jj|)
void soc(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, double theta, uint8_t* strong,
         cudaStream_t s);

// Aggregate (readings c2/c3): priority-order standard aggregation computed as
// MIS-2 rounds + membership + leftover pass.  Returns n_agg; agg[i] in [0, n_agg).
int32_t aggregate(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, const uint8_t* strong,
                  uint64_t seed, int level, int32_t* agg, cudaStream_t s);

// Greedy first-fit colouring in priority order (reading c5) by Jones-Plassmann rounds.
int32_t colour(int32_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed, int32_t* colours, cudaStream_t s);

// Level 0 as A = H H^T + diag(at) (reading c14) for the bootstrap sweeps: fp64 gradients h (m x kc x 3),
// constraint vertices, the vertex -> incidence lists, at = alpha/dt^2 and 1/A_ii.
struct GsOperator {
    int kc = 0;
    int32_t nv = 0;
    const int32_t* verts = nullptr;
    const double* h = nullptr;
    const int64_t* vptr = nullptr;
    const int32_t* vlist = nullptr;
    const double* at = nullptr;
    const double* dinv = nullptr;
};

// Near-kernel bootstrap: `sweeps` colour-major GS sweeps on A x = 0.  With `op` the
// sweeps run matrix-free: u_v = sum_{j at v} h_{j,v} x_j is kept current, row i of a colour reads
// (A x)_i = sum_s h_{i,s}.u_{v_s} + at_i x_i, sets x_i -= (A x)_i / A_ii and adds h_{i,s} dx_i to its
// vertices' u — rows of one colour share no vertex (they are not coupled in A), so the updates are
// race-free and the result is Gauss-Seidel's (rounding aside) at ~1/4 of the CSR sweep's bytes.  The
// CSR values still give x_0's scale max |A_ij| (reading c0).
// idx_offset: the hash index of x_0[i] is i + idx_offset (column c of a k > 1 bootstrap: c n, reading c23).
void gs_bootstrap(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, const int32_t* colours,
                  int32_t ncolours, int32_t sweeps, uint64_t seed, double* B, cudaStream_t s,
                  const GsOperator* op = nullptr, uint64_t idx_offset = 0);

// Inject (k = 1): P_i = B_i / ||B_agg(i)||, B_next[a] = ||B_a|| (members ascending).
void prolongator(int32_t n_agg, const int64_t* mptr, const int32_t* mlist, const double* B, double* P,
                 double* B_next, cudaStream_t s);

// Galerkin symbolic structures for fine level -> coarse level.
struct GalerkinPlan {
    DBuf<uint16_t> gperm;   // per fine nnz: row-relative entry index at sorted position (agg(col), col)
    DBuf<int64_t> tptr;     // fine rows + 1: first t-entry (segment) of each row
    DBuf<int64_t> tstart;   // T + 1: absolute sorted position where segment t starts
    DBuf<int32_t> trow;     // T: fine row of segment t
    DBuf<int32_t> tagg;     // T: coarse column of segment t
    DBuf<int64_t> lptr;     // coarse nnz + 1: ranges into llist
    DBuf<int32_t> llist;    // T: segments grouped by coarse nnz, ascending
    int64_t T = 0;
};

// Builds plan + coarse pattern (crowptr/ccol, off-diagonals ascending, diagonal last).
void galerkin_symbolic(int32_t n, const int64_t* rowptr, const int32_t* col, const int32_t* agg,
                       const int64_t* mptr, const int32_t* mlist, int32_t n_agg, GalerkinPlan& plan,
                       DBuf<int64_t>& crowptr, DBuf<int32_t>& ccol, cudaStream_t s);

// Numeric Galerkin (Eq. 6): cval = P^T A P over the cached plan; cdinv = 1/diag.
template <class T>
void galerkin_numeric(const GalerkinPlan& plan, const int64_t* rowptr, const int32_t* col, const T* val,
                      const T* P, int32_t n_agg, const int64_t* crowptr, int64_t cnnz, T* tval, T* cval, T* cdinv,
                      cudaStream_t s, int64_t t_begin = 0, int64_t t_end = -1);
// (segments [t_begin, t_end) only — the others keep their tval; cdinv == nullptr skips 1/diag)

template <class T>
void diag_inv(int32_t n, const int64_t* rowptr, const T* val, T* dinv, cudaStream_t s);

// lambda_max(D^-1 A) by the power method (reading c9); returns lambda (host sync).
// Same iteration with the operator given as apply(v, w, parts): w = D^-1 A v and the partials of
// |w|^2; returns the number of partials written.  (Level 0 uses the matrix-free operator.)
// init = false: start from the normalised vector already in v (the per-frame omega refresh, reading c26).
// On return v holds the last normalised iterate.
double power_method_op(int32_t n, int dot_grid, const std::function<int(const double*, double*, double*)>& apply,
                       int32_t iters, uint64_t seed, int level, double* v, double* w, double* parts, double* ss,
                       cudaStream_t s, bool init = true);
double power_method(const Csr<double>& A, int32_t iters, uint64_t seed, int level, double* v, double* w,
                    double* parts, double* ss, cudaStream_t s, bool init = true);

}  // namespace mgpbd
