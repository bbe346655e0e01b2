// Constraint-side kernels: rest data, vertex incidence, fixed CSR pattern, constraint evaluation,
// numeric re-assembly, predict and position update.
#pragma once
#include "common.cuh"

namespace mgpbd {

void rest_distance(const int32_t* verts, const double* X, int32_t m, double* L, cudaStream_t s);
void rest_arap(const int32_t* verts, const double* X, int32_t m, double* Dminv, double* vol,
               int32_t* bad, cudaStream_t s);

// vertex -> (constraint*kc + slot) lists, ascending per vertex
void build_incidence(const int32_t* verts, int32_t m, int kc, int32_t nv, DBuf<int64_t>& vptr,
                     DBuf<int32_t>& vlist, cudaStream_t s);

// Fixed CSR pattern of A: row i = sorted constraints sharing a vertex with i, then i.
void build_pattern(const int32_t* verts, int32_t m, int kc, int32_t nv, const int64_t* vptr,
                   const int32_t* vlist, DBuf<int64_t>& rowptr, DBuf<int32_t>& col, cudaStream_t s);

// Constraint evaluation (Alg. 1 l.4 + l.6): scaled gradients h = sqrt(w) grad C and b = -C - at*lambda.
// EvalHv (optional, one rank, every row): the kernel also writes the matrix-free operator's per-outer-iteration data
// that k_mf_refresh would build from h — the vertex-major planes hv[plane npad + inv[j kc + k]] = h_{j,k,plane}
// (inv: padded slot of incidence (j, k)), at_j = alpha_j / dt^2 and dinv_j with k_mf_refresh's expression.
template <class T>
struct EvalHv {
    const int32_t* inv = nullptr;
    T* hv = nullptr;
    int64_t npad = 0;
    T* at = nullptr;
    T* dinv = nullptr;
};
template <class T>
void eval_constraints(int kind, int32_t m, const int32_t* verts, const double* x, const double* rest,
                      const double* sqrtw, const double* alpha, double dt, const double* lambda,
                      T* h, T* b, cudaStream_t s, const EvalHv<T>* hvout = nullptr);

// Numeric re-assembly (Alg. 1 l.5) into the fixed pattern; also dinv = 1/A_ii.
template <class T>
void assemble(int kind, int32_t m, const int32_t* verts, const T* h, const double* alpha, double dt,
              const int64_t* rowptr, const int32_t* col, int vl, T* val, T* dinv, cudaStream_t s, int32_t row0 = 0,
              int32_t row1 = -1);  // rows [row0, row1) (default: all m)

void predict(int32_t n, double* x, double* v, double* x_old, const double* w, double dt,
             double gx, double gy, double gz, cudaStream_t s);
template <class T>
void update_positions(int32_t n, int kc, const int64_t* vptr, const int32_t* vlist, const T* h,
                      const double* sqrtw, const T* dl, const double* omega, double* x, cudaStream_t s);
template <class T>
void lambda_add(int32_t m, double* lambda, const T* dl, cudaStream_t s);
// omega *= 1/2 (>= omega_min) if ||b_ite||^2 > ||b_{ite-1}||^2 (device scalars; reading c21)
void backtrack_omega(const double* bn2, int ite, double* omega, double omega_min, cudaStream_t s);
void velocity(int32_t n, const double* x, const double* x_old, double* v, double dt, cudaStream_t s);
void sqrt_vec(int32_t n, const double* w, double* out, cudaStream_t s);

}  // namespace mgpbd
