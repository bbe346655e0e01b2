// Hot-loop kernels: fused CSR passes (omega-Jacobi sweep, residual*P, SpMV+dot, power step),
// aggregate restriction, prolongation, PCG vector updates, coarsest dense inverse + GEMV
// (SURVEY.md §8(a) rows a8-a11).
#pragma once
#include "common.cuh"

namespace mgpbd {

template <class T>
struct Csr {
    int32_t row0 = 0;  // first row processed (global index); rows [row0, row0 + n)
    int32_t n = 0;
    int64_t nnz = 0;
    const int64_t* rowptr = nullptr;
    const int32_t* col = nullptr;
    const T* val = nullptr;
    const T* dinv = nullptr;
    int vl = 32;     // lanes per row (warp-per-row kernel)
    int grid = 1;    // fixed grid (=> fixed partial count => deterministic reductions)
    int nparts = 1;  // number of per-CTA partials a dot-producing pass writes
    int vlr = 0;     // > 0: row-tile kernel with 256/vlr rows per tile and vlr reduce lanes per row
    int tile_nnz = 0;  // max nnz of a tile (shared-memory products)
    // band-staged kernel (band_rows > 0): band tiles of band_rows rows, x window per band tile
    int band_rows = 0, band_grid = 0, prod_cap = 0, band_win = 0;
    int row_vl = 0;  // > 0: barrier-free band row kernel with row_vl lanes per row
    const int32_t* win_lo = nullptr;
    const int32_t* win_len = nullptr;
    const uint16_t* col16 = nullptr;  // window-relative column offsets (hot copy, row kernel)
};

// Band configuration for the band-staged pass: returns false (and C = 0) if the column window of even
// the smallest band tile does not fit in shared memory next to the product buffer.  With the row
// kernel (row_vl > 0) it also builds col16, the 16-bit window-relative copy of the column indices.
template <class T>
bool band_config(int32_t row0, int32_t n, const int64_t* rowptr, const int32_t* col, int vlr, DBuf<int32_t>& lo,
                 DBuf<int32_t>& len, int& C, int& grid, int& prod_cap, int& win, int& row_vl, DBuf<uint16_t>& col16,
                 cudaStream_t s);

// PCG scalar commit for a partitioned solve: d2 = (r.z, r.r) or d1 = (p.q) already summed over ranks.
void pcg_commit_rz(const double* d2, double* scal, int k, int* flags, int tag, cudaStream_t s);
// PCG scalar slots of `scal` (2 * 4096 doubles; iteration k uses 2k, 2k + 1 for k < SC_KMAX): the
// optional convergence exit (pcg_tol > 0): tolerance, ||b||^2, and the "converged" flag that freezes
// the remaining iterations (their updates are skipped, so the result equals an early exit).
constexpr int SC_KMAX = 4090;
constexpr int SC_TOL = 8189, SC_B2 = 8190, SC_DONE = 8191;
void pcg_begin(double* scal, double tol, cudaStream_t s);
// flags[7] = outer-iteration index (written eagerly before each outer iteration, so the captured
// iteration graph is the same for every ite; the flag kernels report ite * 4096 + pcg iteration)
void set_outer_index(int* flags, int ite, cudaStream_t s);
void pcg_commit_pq(const double* d1, double* scal, int k, int* flags, int tag, cudaStream_t s);

// Column window [min col, max col] referenced by rows [a, b) (diagonal-last CSR); host result.
void row_range_window(const int64_t* rowptr, const int32_t* col, int32_t a, int32_t b, int32_t* lo, int32_t* hi,
                      cudaStream_t s);

// Choose the row-tile configuration of a level (vlr, fixed grid, max tile nnz); vlr = 0 if the tile
// would not fit in shared memory.
void tile_config(int32_t n, int64_t nnz, const int64_t* rowptr, int& vlr, int& grid, int& tile_nnz, cudaStream_t s);

enum PassMode {
    PASS_JACOBI = 0,      // y = x + omega dinv (b - A x)
    PASS_JACOBI_DOT = 1,  // same, plus partials of sum aux_i*y_i and sum aux_i^2 (aux = PCG r)
    PASS_RESID_P = 2,     // y = aux * (b - A x)   (aux = P: restriction input)
    PASS_SPMV_DOT = 3,    // y = A x, partials of sum x_i*y_i
    PASS_POWER = 4,       // y = dinv (A x), partials of sum y_i^2
    PASS_JACOBI0_FIRST = 5
};

int pass_grid(int32_t n, int vl);

template <class T>
void csr_pass(int mode, const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega,
              double* parts, double* parts2, cudaStream_t s, double alpha = 0.0, const T* xprev = nullptr);
// (PASS_JACOBI / PASS_JACOBI_DOT with alpha != 0: y = x + alpha (x - xprev) + omega D^-1 (b - A x),
//  the Chebyshev three-term step; xprev == nullptr means xprev = 0)

template <class T> void vec_jacobi0(int32_t n, const T* dinv, const T* b, double omega, T* y, cudaStream_t s);
template <class T> void restrict_members(int32_t nc, const int64_t* mptr, const int32_t* mlist, const T* t,
                                         T* bc, cudaStream_t s);
template <class T> void prolong_add(int32_t n, const int32_t* agg, const T* P, const T* e, T* x, cudaStream_t s);
// p = z + beta p with beta = rz[k]/rz[k-1] (0 if k == 0 or rz[k-1] == 0)
template <class T> void pcg_update_p(int32_t n, const T* z, T* p, const double* scal, int k, cudaStream_t s);
// one multicolour Gauss-Seidel sweep in place (colours 0..ncol-1, or reversed), rows grouped by colour
template <class T>
void gs_sweep(const Csr<T>& A, const int64_t* gs_ptr, const int32_t* gs_list, int ncol, bool backward, const T* b, T* x,
              cudaStream_t s);
// single-GPU variants with the dot finalisation fused in (same flags / scal semantics as the
// pcg_finalize_* + pcg_update_* pairs)
template <class T>
void pcg_update_p_fin(int32_t n, const T* z, T* p, double* scal, int k, const double* prz, const double* prr, int np,
                      int* flags, int tag, cudaStream_t s, const double* fin = nullptr);
template <class T>
void pcg_update_xr_fin(int32_t n, const T* p, const T* q, T* x, T* r, double* scal, int k, const double* ppq, int np,
                       int* flags, int tag, cudaStream_t s, const T* dinv = nullptr, double om0 = 0.0, T* x1 = nullptr,
                       const double* fin = nullptr);
// (fin != nullptr: the partial sums were already summed by the producing matrix-free row kernel, MatFree::fin)
// (x1 != nullptr: also x1 = om0 D^-1 r_new, the next V-cycle's first smoothing step from x = 0)
// alpha = rz[k]/pq[k] (0 if pq == 0); x += alpha p; r -= alpha q
template <class T> void pcg_update_xr(int32_t n, const T* p, const T* q, T* x, T* r, const double* scal, int k,
                                      cudaStream_t s);
template <class T> void dot_parts(int32_t n, const T* a, const T* b, double* parts, int grid, cudaStream_t s);
// power method normalisation: v = w / sqrt(scal[0])
template <class T> void scale_by_inv_sqrt(int32_t n, const T* w, T* v, const double* ss, cudaStream_t s);

// PCG scalar layout in the device scalar array: rz[k] at 2k, pq[k] at 2k+1; flags int array:
// flags[0] indefinite, flags[1] non-finite (first occurrence iteration in flags[2..3]).
void pcg_finalize_rz(const double* parts_rz, const double* parts_rr, int np, double* scal, int k, int* flags,
                     int tag, cudaStream_t s);
void pcg_finalize_pq(const double* parts, int np, double* scal, int k, int* flags, int tag, cudaStream_t s);

// Coarsest level: dense inverse by Gauss-Jordan (SPD, no pivoting; reading c8) of the CSR values,
// then GEMV x = Ainv b.
template <class T>
void coarse_invert(const Csr<T>& A, double* work, double* Ainv, int* flags, cudaStream_t s);
template <class T> void coarse_gemv(int32_t n, const double* Ainv, const T* b, T* x, cudaStream_t s);

}  // namespace mgpbd
