// The coarse part of the V-cycle (levels l >= 1) as ONE persistent cooperative
// kernel with grid-wide barriers between dependent phases, instead of ~7 launches per level.
//
// Below level 0 every level is small (block1.67M: 71K, 17K, 4.9K, 2K, 804, 357 rows) and the
// multi-kernel V-cycle is bound by launch gaps and tails, not by bytes.  Phases per level (nu = 2):
//   down: [omega-Jacobi sweep 2 with sweep 1 (x = omega D^-1 b) evaluated on the fly]  | barrier
//         [residual * P and restriction, aggregate-major: r_i, t_i = P_i r_i, sum over members] | barrier
//   coarsest: z = A_c^-1 b (dense fp64 inverse)                                          | barrier
//   up:   [sweep 1 with the prolongation x_j + P_j z_c[agg_j] evaluated on the fly]      | barrier
//         [sweep 2 -> z]                                                                  | barrier
// Smoother steps are the general x_{k+1} = x_k + alpha_k (x_k - x_{k-1}) + omega_k D^-1 (b - A x_k)
// (omega-Jacobi: alpha = 0; Chebyshev: three-term recurrence).
// Same operators, smoothing schedule and arithmetic precision as the per-level kernels (solve.cu);
// only the summation order inside a row differs.
#pragma once
#include "common.cuh"

namespace mgpbd {

template <class T>
struct CoarseLevel {
    int32_t n = 0;
    const int64_t* rowptr = nullptr;
    const int32_t* col = nullptr;
    const T* val = nullptr;
    const T* dinv = nullptr;
    double omega = 0.0;             // (unused by the cycle; the per-step coefficients below)
    // smoother step k (k < nu): x_{k+1} = x_k + alpha_k (x_k - x_{k-1}) + omega_k D^-1 (b - A x_k);
    // omega-Jacobi: omega_k = omega, alpha_k = 0; Chebyshev: the three-term recurrence (reading c20)
    double sm_omega[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double sm_alpha[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // towards the next level (unused on the coarsest)
    const int32_t* agg = nullptr;
    const T* P = nullptr;
    const int64_t* mptr = nullptr;
    const int32_t* mlist = nullptr;
    int32_t n_agg = 0;
    // vectors: rhs b, result z, scratch x / y, restriction input t
    T* t = nullptr;
    T* b = nullptr;
    T* z = nullptr;
    T* x = nullptr;
    T* y = nullptr;
};

template <class T>
struct CoarseCycle {
    int K = 0;                    // levels in the cycle (the last is the coarsest)
    int nu = 2;                   // pre = post sweeps
    const double* Ainv = nullptr; // coarsest dense inverse (n_{K-1}^2, fp64)
    unsigned long long* trace = nullptr;  // optional: %globaltimer after each phase (block 0), 64 slots
    CoarseLevel<T> L[16];
};

// z_0 = V(b_0) over levels 0..K-1 of `c` (x = 0 start on every level).  One launch.
template <class T>
void coarse_vcycle(const CoarseCycle<T>& c, cudaStream_t s);

}  // namespace mgpbd
