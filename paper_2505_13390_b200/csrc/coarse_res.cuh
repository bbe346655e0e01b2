// Shared-memory-resident variant of the persistent coarse V-cycle (coarse.cuh).
//
// One CTA per SM owns a contiguous, nnz-balanced row range of every coarse level and a member-balanced
// aggregate range; at kernel start it copies its slices of the static data (CSR offsets, columns and
// values, D^-1, P, aggregate ids, member lists, its rows of the coarsest inverse) into shared memory
// with 1-D bulk copies.  Every phase then reads the matrix from shared memory and only gathers vectors
// from L2: one dependent round trip per row wave instead of two.  Used when the slices fit (the block
// hierarchies do); otherwise the global-memory kernel runs.
#pragma once
#include <vector>

#include "coarse.cuh"
#include "coarse_tail.cuh"

namespace mgpbd {

struct ResLevel {        // one CTA's share of one coarse level
    int32_t r0 = 0, r1 = 0;  // owned rows
    int32_t a0 = 0, a1 = 0;  // owned aggregates (towards the next level)
    int64_t e0 = 0;          // rowptr[r0]
    int64_t m0 = 0;          // mptr[a0]
    // shared-memory byte offsets of element r0 / e0 / a0 / m0 of each slice
    uint32_t o_rp = 0, o_col = 0, o_val = 0, o_dinv = 0, o_P = 0, o_agg = 0, o_mp = 0, o_ml = 0;
};
struct ResCopy {
    const void* src;     // 16-byte aligned
    uint32_t dst;        // shared-memory byte offset, 16-byte aligned
    uint32_t bytes;      // multiple of 16; bit 31 (RES_LATE): a copy of cycle level >= 1 (second barrier)
};
constexpr uint32_t RES_LATE = 0x80000000u;
constexpr uint32_t RES_BYTES_MASK = 0x7fffffffu;

constexpr int RES_MAXC = 128;  // bulk copies per CTA

// "Solo" tail: the smallest levels (cycle levels solo_first..K-1, the coarsest inverse included) held whole in
// CTA 0's shared memory and cycled by that CTA alone with __syncthreads between phases while the other CTAs
// wait at one grid barrier — no grid barrier per phase.  Offsets are CTA-0 shared-memory byte offsets of
// element 0 of each whole-level array.
struct SoloLevel {
    int32_t n = 0;
    uint32_t o_rp = 0, o_col = 0, o_val = 0, o_dinv = 0, o_P = 0, o_agg = 0, o_mp = 0, o_ml = 0;
    uint32_t o_b = 0, o_x = 0, o_y = 0, o_t = 0, o_z = 0;   // vectors (not copied)
};
constexpr int SOLO_MAXL = 8;

struct ResPlan {
    int G = 0;                       // CTAs (one per SM)
    uint32_t smem = 0;               // dynamic shared memory per CTA
    const ResLevel* lv = nullptr;    // [G][16]
    const ResCopy* copies = nullptr; // [G][RES_MAXC]
    const int32_t* ncopies = nullptr;
    const uint32_t* txbytes = nullptr;
    int solo_first = 0;              // > 0: cycle levels solo_first..K-1 run on CTA 0 alone (mode 0)
    SoloLevel solo[SOLO_MAXL];
};

// Host: build the plan for cycle `c` (host copies of each level's rowptr / mptr are downloaded).
// Returns false if some CTA's slices exceed `smem_cap` bytes (then the global kernel is used).
// with_coarsest = false: the last level of `c` gets no slices (the cycle is split around the cluster tail,
// coarse_tail.cuh, whose first level is c's last).
// solo = true: also plan the solo tail (the longest suffix of levels, at least one above the coarsest, whose
// whole data fits CTA 0 next to its slices); plan.solo_first / plan.solo are filled through *solo_out.
template <class T>
bool coarse_res_plan(const CoarseCycle<T>& c, int G, uint32_t smem_cap, std::vector<ResLevel>& lv,
                     std::vector<ResCopy>& copies, std::vector<int32_t>& ncopies, std::vector<uint32_t>& tx,
                     uint32_t& smem, cudaStream_t s, bool with_coarsest = true, ResPlan* solo_out = nullptr);

// mode 0: the whole cycle; 1: down phase of levels 0..kstop-1 (leaves b of level kstop); 2: up phase from
// level kstop-1 (reads z of level kstop); 3: 1 + the cluster tail (coarse_tail.cuh) on the launch's first
// cluster + 2, in ONE cooperative launch with cluster dimensions (tail: its arguments, its shared-memory
// region at tail_base of tail_smem bytes).
template <class T>
void coarse_vcycle_res(const CoarseCycle<T>& c, const ResPlan& plan, cudaStream_t s, int mode = 0, int kstop = 0,
                       const TailArgs<T>* tail = nullptr, uint32_t tail_base = 0, uint32_t tail_smem = 0);
// co-resident CTAs of the mode-3 launch in clusters of CT with `smem` bytes (multiple of CT; 0: none)
template <class T>
int coarse_res_fused_grid(int CT, uint32_t smem);
// CTAs of k_coarse_vcycle_res<T> that fit on one SM with `smem` dynamic bytes (0: the resident plan
// cannot be launched cooperatively at one CTA per SM; the caller falls back to the global kernel)
template <class T>
int coarse_res_blocks_per_sm(uint32_t smem);

}  // namespace mgpbd
