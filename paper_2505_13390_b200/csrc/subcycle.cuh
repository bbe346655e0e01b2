// The bottom of the V-cycle as one dense operator (reading c27).
//
// From a level l_c down, the V-cycle of PAPER.md:313-318 started from x = 0 is a fixed LINEAR map of its
// right-hand side: z_{l_c} = M b_{l_c}, with M determined by the level matrices, P, the aggregates, the
// smoother coefficients and the coarsest inverse.  When n_{l_c} is small (<= ~1000 rows) the hot cycle
// applies M as one dense GEMV instead of the ~7 latency-bound barrier phases of levels l_c..L-1;
// M is rebuilt whenever those levels change (every Eq. 6 refresh, i.e. every outer iteration) by running
// the same sub-cycle on the unit vectors e_j: CTAs take blocks of CB columns, keep the level vectors of
// their columns in shared memory (one thread per (row, column) pair, the level CSR read from L2, row sums
// in fp64) and write M row-major in fp64, like the coarsest inverse it extends (reading c8).  Same
// arithmetic as the hot cycle's sweeps / residual / restriction / prolongation up to rounding.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace mgpbd {

constexpr int SUB_MAXL = 8;

template <class T>
struct SubLevel {
    int32_t n = 0;
    const int64_t* rowptr = nullptr;
    const int32_t* col = nullptr;
    const T* val = nullptr;        // diagonal last in every row
    const T* dinv = nullptr;
    double om[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // smoother step coefficients (engine set_smoother)
    double al[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // towards the next level (unused on the coarsest)
    const int32_t* agg = nullptr;
    const T* P = nullptr;
    const int64_t* mptr = nullptr;
    const int32_t* mlist = nullptr;
    int32_t nnz = 0, n_next = 0;   // entries; rows of the next level (= aggregates)
    // shared-memory element offsets (units of T, per column block) of this level's b and pre-smoothed x
    uint32_t o_b = 0, o_xs = 0;
    // staged copies (byte offsets; SubCycle::staged): rowptr / mptr as int32, col, val, dinv, P, agg, mlist
    uint32_t s_rp = 0, s_col = 0, s_val = 0, s_dinv = 0, s_P = 0, s_agg = 0, s_mp = 0, s_ml = 0;
};

template <class T>
struct SubCycle {
    int K = 0;                    // levels l_c..L-1 (the last is the coarsest)
    int nu = 2;                   // pre = post smoothing steps
    const double* Ainv = nullptr; // coarsest inverse, row-major n_{K-1}^2
    uint32_t o_s0 = 0, o_s1 = 0, o_s2 = 0;  // three scratch vectors (max n each)
    uint32_t smem = 0;            // dynamic shared memory bytes per CTA
    bool staged = false;          // the level CSR / P / aggregates / members and Ainv copied into shared memory
    uint32_t s_ainv = 0;          // byte offset of the staged Ainv
    uint32_t vec_bytes = 0;       // bytes of the vector section (offset of the staged data)
    SubLevel<T> L[SUB_MAXL];
};

// Host: fill the shared-memory layout of `c` (levels already set); false if it exceeds `cap` bytes.
template <class T>
bool subcycle_plan(SubCycle<T>& c, uint32_t cap);

// M (n_0 x n_0, row-major fp64) = the sub-cycle applied to every unit vector.
template <class T>
void subcycle_matrix(const SubCycle<T>& c, double* M, cudaStream_t s);

}  // namespace mgpbd
