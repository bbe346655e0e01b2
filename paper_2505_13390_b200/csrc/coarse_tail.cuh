// The smallest coarse levels of the V-cycle on ONE thread-block cluster.
//
// Below a few thousand rows a V-cycle phase is pure latency: on the grid-wide persistent kernel every
// phase pays a grid barrier (~1.2 us) plus a dependent L2 round trip for the vector gathers, ~3-4.5 us per
// phase for levels of 357..4915 rows.  Here the tail levels j..K-1 run on one cluster of
// CT (16, else 8) CTAs, one per SM:
//   * each CTA holds its own rows of every tail level (CSR with 16-bit column indices, D^-1, P, aggregate
//     ids), its rows of the coarsest dense inverse and the member-slot ranges of its own aggregates in
//     shared memory (bulk copies at kernel start);
//   * every CTA keeps FULL copies of each tail level's vectors (two ping-pong buffers): a phase computes
//     its own rows and broadcasts them into all CTAs' copies through distributed shared memory, so the
//     next phase gathers from local shared memory only;
//   * phases are separated by barrier.cluster (~0.2 us) instead of grid barriers;
//   * restriction: the aggregate owner (= the owner of that row on the next level) receives each member's
//     residual*P into a slot array (one DSMEM store per row) and sums its members in ascending order.
// Operators, smoothing schedule and precision are those of the grid-wide kernel (coarse.cuh); only the
// summation order inside a row (8-lane butterfly) is shared with it.  The levels above j stay on the
// grid-wide kernel, split around this one (coarse_res.cuh: down phase, tail, up phase).
#pragma once
#include <vector>

#include "coarse.cuh"

namespace mgpbd {

constexpr int TAIL_MAXL = 8;      // levels in the tail (the last is the coarsest)
constexpr int TAIL_MAXC = 64;     // bulk copies per CTA

struct TailLevel {                // one CTA's share of one tail level (smem byte offsets)
    int32_t n = 0;                // rows of the level
    int32_t r0 = 0, r1 = 0;       // own rows
    int32_t a0 = 0, a1 = 0;       // own aggregates towards the next level (= own rows there)
    int64_t e0 = 0;               // rowptr[r0]
    int64_t m0 = 0;               // mptr[a0]
    uint32_t o_rp = 0, o_col = 0, o_val = 0, o_dinv = 0, o_P = 0, o_agg = 0, o_push = 0, o_mp = 0;
    uint32_t o_slot = 0, o_b = 0, o_X = 0, o_Y = 0, o_Ainv = 0;
    uint32_t ob = 0;              // bulk broadcast: bytes of this CTA's own rows (16-byte multiple)
    uint32_t rx = 0;              //   and the bytes it receives from the other CTAs per broadcast
};
struct TailCopy {
    const void* src;
    uint32_t dst, bytes;
};

template <class T>
struct TailArgs {
    int KT = 0;                        // tail levels (last = coarsest)
    int nu = 2;
    int CT = 16;                       // CTAs in the cluster
    const TailLevel* lv = nullptr;     // [CT][TAIL_MAXL]
    const TailCopy* copies = nullptr;  // [CT][TAIL_MAXC]
    const int32_t* ncopies = nullptr;
    const uint32_t* txbytes = nullptr;
    const T* b_top = nullptr;          // rhs of the first tail level (global, written by the down phase)
    T* z_top = nullptr;                // its V-cycle result (global, read by the up phase)
    double sm_omega[TAIL_MAXL][8];
    double sm_alpha[TAIL_MAXL][8];
    unsigned long long* trace = nullptr;
    int bulk = 0;                      // 1: broadcasts as cp.async.bulk shared::cta -> shared::cluster copies
};

struct TailPlan {
    int first = 0;                     // cycle index of the first tail level (levels first..K-1)
    int CT = 0;
    int bulk = 0;                      // row ranges 16-byte aligned: bulk DSMEM broadcasts
    uint32_t smem = 0;
    DBuf<TailLevel> lv;
    DBuf<TailCopy> copies;
    DBuf<int32_t> ncopies;
    DBuf<uint32_t> txbytes;
    DBuf<uint16_t> col16[TAIL_MAXL];    // per tail level (non-coarsest): 16-bit column indices
    DBuf<int32_t> push[TAIL_MAXL];      // per tail level: destination (cta << 24 | slot offset) of row i's t_i
};

// Host: plan levels [first, K) of `c` on one cluster of CT CTAs; false if no first >= min_first fits
// `smem_cap` bytes per CTA (then the grid-wide kernel keeps every level).
template <class T>
bool coarse_tail_plan(const CoarseCycle<T>& c, int min_first, int CT, uint32_t smem_cap, TailPlan& plan, cudaStream_t s);

// CTs the device can run as one cluster with `smem` bytes and the tail kernel's block (0: none).
template <class T>
bool coarse_tail_launchable(int CT, uint32_t smem);

// z_first = V(b_first) over the tail levels.
template <class T>
void coarse_tail_run(const CoarseCycle<T>& c, const TailPlan& plan, cudaStream_t s);
// The kernel arguments of the tail (for the fused grid + cluster kernel, coarse_res.cuh mode 3).
template <class T>
TailArgs<T> coarse_tail_args(const CoarseCycle<T>& c, const TailPlan& plan);

}  // namespace mgpbd
