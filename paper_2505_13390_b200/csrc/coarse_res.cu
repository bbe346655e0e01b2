// Shared-memory-resident persistent coarse V-cycle, see coarse_res.cuh.
#include <cooperative_groups.h>

#include <algorithm>

#include "coarse_res.cuh"
#include "coarse_tail_body.cuh"
#include "comm.cuh"
#include "tma.cuh"
#include "util.cuh"

namespace cg = cooperative_groups;

namespace mgpbd {

namespace {

#ifndef MGPBD_RES_SVL
#define MGPBD_RES_SVL 8
#endif
#ifndef MGPBD_RES_SCH
#define MGPBD_RES_SCH 5
#endif
constexpr int RB = 1024;  // threads per CTA (one CTA per SM)
constexpr int RSVL = MGPBD_RES_SVL;   // lanes per row (build switch, sweeps)
constexpr int RSCH = MGPBD_RES_SCH;   // nonzeros per lane per chunk
constexpr int RRPW = 32 / RSVL;
constexpr int RCHUNK = RSVL * RSCH;
constexpr int RWARPS = RB / 32;

// one CTA's slices of one level in shared memory (offsets point at element r0 / e0 / a0 / m0)
template <class T>
struct Slice {
    const unsigned char* sm;
    ResLevel d;
    __device__ int64_t rp(int64_t i) const { return reinterpret_cast<const int64_t*>(sm + d.o_rp)[i - d.r0]; }
    __device__ int32_t col(int64_t e) const { return reinterpret_cast<const int32_t*>(sm + d.o_col)[e - d.e0]; }
    __device__ T val(int64_t e) const { return reinterpret_cast<const T*>(sm + d.o_val)[e - d.e0]; }
    __device__ T dinv(int64_t i) const { return reinterpret_cast<const T*>(sm + d.o_dinv)[i - d.r0]; }
    __device__ T P(int64_t i) const { return reinterpret_cast<const T*>(sm + d.o_P)[i - d.r0]; }
    __device__ int32_t agg(int64_t i) const { return reinterpret_cast<const int32_t*>(sm + d.o_agg)[i - d.r0]; }
    __device__ int64_t mp(int64_t a) const { return reinterpret_cast<const int64_t*>(sm + d.o_mp)[a - d.a0]; }
    __device__ int32_t ml(int64_t e) const { return reinterpret_cast<const int32_t*>(sm + d.o_ml)[e - d.m0]; }
    __device__ const double* dense_rows() const { return reinterpret_cast<const double*>(sm + d.o_val); }
};

struct Lanes {
    int lane, sub, sl, warp;
    __device__ Lanes() {
        lane = threadIdx.x & 31;
        sub = lane / RSVL;
        sl = lane % RSVL;
        warp = threadIdx.x >> 5;
    }
};

// sum_k A_ik x(col_k) for row i (owned by this CTA; matrix from shared memory); warp-wide butterfly
template <class T, class XF>
__device__ __forceinline__ double row_sum(const Lanes& w, const Slice<T>& S, bool valid, int64_t i, XF xf) {
    const int64_t a = valid ? S.rp(i) : 0, e = valid ? S.rp(i + 1) : 0;
    const int maxlen = __reduce_max_sync(0xffffffffu, (int)(e - a));
    T part = (T)0;
    for (int off = 0; off < maxlen; off += RCHUNK) {
        int32_t c[RSCH];
        T v[RSCH], xv[RSCH];
#pragma unroll
        for (int q = 0; q < RSCH; ++q) {
            const int64_t k = a + off + q * RSVL + w.sl;
            const bool in = k < e;
            c[q] = in ? S.col(k) : -1;
            v[q] = in ? S.val(k) : (T)0;
        }
#pragma unroll
        for (int q = 0; q < RSCH; ++q) xv[q] = c[q] >= 0 ? xf(c[q]) : (T)0;
#pragma unroll
        for (int q = 0; q < RSCH; ++q) part += v[q] * xv[q];
    }
    return (double)group_sum_t<RSVL>(part);
}

// smoother step over this CTA's rows: y = x + alpha (x - xprev) + omega D^-1 (b - A x)
template <class T, class XF, class XPF>
__device__ __forceinline__ void sweep(const Lanes& w, const CoarseLevel<T>& L, const Slice<T>& S, XF xf, XPF xpf,
                                      double omega, double alpha, T* __restrict__ out) {
    for (int64_t base = S.d.r0 + w.warp * RRPW; base < S.d.r1; base += RWARPS * RRPW) {  // warp-uniform
        const int64_t i = base + w.sub;
        const bool valid = i < S.d.r1;
        const double s = row_sum(w, S, valid, i, xf);
        if (valid && w.sl == 0) {
            const double xi = (double)xf((int32_t)i);
            double y = xi + omega * (double)S.dinv(i) * ((double)L.b[i] - s);
            if (alpha != 0.0) y += alpha * (xi - (double)xpf((int32_t)i));
            out[i] = (T)y;
        }
    }
}

template <class T>
__device__ __forceinline__ void resid(const Lanes& w, const CoarseLevel<T>& L, const Slice<T>& S,
                                      const T* __restrict__ x) {
    for (int64_t base = S.d.r0 + w.warp * RRPW; base < S.d.r1; base += RWARPS * RRPW) {
        const int64_t i = base + w.sub;
        const bool valid = i < S.d.r1;
        const double s = row_sum(w, S, valid, i, [&](int32_t j) { return x[j]; });
        if (valid && w.sl == 0) L.t[i] = (T)((double)S.P(i) * ((double)L.b[i] - s));
    }
}

template <class T>
__device__ __forceinline__ void restrict_t(const Lanes& w, const CoarseLevel<T>& L, const Slice<T>& S,
                                           T* __restrict__ bnext) {
    for (int64_t base = S.d.a0 + w.warp * RRPW; base < S.d.a1; base += RWARPS * RRPW) {
        const int64_t a = base + w.sub;
        double s = 0.0;
        if (a < S.d.a1) {
            const int64_t m1 = S.mp(a + 1);
            for (int64_t e = S.mp(a) + w.sl; e < m1; e += RSVL) s += (double)L.t[S.ml(e)];
        }
        s = group_sum<RSVL>(s);
        if (a < S.d.a1 && w.sl == 0) bnext[a] = (T)s;
    }
}

template <class T>
__device__ __forceinline__ void dense_solve(const Lanes& w, int32_t n, const Slice<T>& S, const T* __restrict__ b,
                                            T* __restrict__ x) {
    const double* A = S.dense_rows();
    for (int64_t i = S.d.r0 + w.warp; i < S.d.r1; i += RWARPS) {
        double s = 0.0;
        for (int32_t j = w.lane; j < n; j += 32) s += A[(i - S.d.r0) * n + j] * (double)b[j];
        s = group_sum<32>(s);
        if (w.lane == 0) x[i] = (T)s;
    }
}

// The solo tail (coarse_res.cuh SoloLevel): cycle levels js..K-1 of `c` by this CTA alone.  Same operators,
// smoothing steps and lane structure (8 lanes per row, fixed butterfly) as the grid phases; reads b of level
// js from global memory and writes its z there.
template <class T>
__device__ void solo_cycle(const Lanes& w, const CoarseCycle<T>& c, const ResPlan& plan, int js, unsigned char* sm) {
    const int K = c.K, nu = c.nu, nl = K - js;
    auto P_ = [&](uint32_t off) { return reinterpret_cast<T*>(sm + off); };
    auto rowsum = [&](const SoloLevel& S, int32_t i, bool valid, const T* x) {
        const int64_t* rp = reinterpret_cast<const int64_t*>(sm + S.o_rp);
        const int32_t* col = reinterpret_cast<const int32_t*>(sm + S.o_col);
        const T* val = reinterpret_cast<const T*>(sm + S.o_val);
        const int64_t a = valid ? rp[i] : 0, e = valid ? rp[i + 1] : 0;
        const int maxlen = __reduce_max_sync(0xffffffffu, (int)(e - a));
        T part = (T)0;
        for (int off = 0; off < maxlen; off += RCHUNK) {
            T v[RSCH], xv[RSCH];
#pragma unroll
            for (int q = 0; q < RSCH; ++q) {
                const int64_t k = a + off + q * RSVL + w.sl;
                const bool in = k < e;
                v[q] = in ? val[k] : (T)0;
                xv[q] = in ? x[col[k]] : (T)0;
            }
#pragma unroll
            for (int q = 0; q < RSCH; ++q) part += v[q] * xv[q];
        }
        return (double)group_sum_t<RSVL>(part);
    };
    // smoother step over all rows: out = x + alpha (x - xprev) + omega D^-1 (b - A x); xprev == nullptr: 0
    auto sweep = [&](const SoloLevel& S, const T* x, const T* xprev, double om, double al, T* out) {
        const T* d = P_(S.o_dinv);
        const T* b = P_(S.o_b);
        for (int32_t base = w.warp * RRPW; base < S.n; base += RWARPS * RRPW) {
            const int32_t i = base + w.sub;
            const bool valid = i < S.n;
            const double sum = rowsum(S, i, valid, x);
            if (valid && w.sl == 0) {
                const double xi = (double)x[i];
                double y = xi + om * (double)d[i] * ((double)b[i] - sum);
                if (al != 0.0) y += al * (xi - (xprev ? (double)xprev[i] : 0.0));
                out[i] = (T)y;
            }
        }
        __syncthreads();
    };
    {   // rhs of the first solo level
        T* b0 = P_(plan.solo[0].o_b);
        for (int32_t i = threadIdx.x; i < plan.solo[0].n; i += blockDim.x) b0[i] = c.L[js].b[i];
        __syncthreads();
    }
    T* curs[SOLO_MAXL];
    for (int t = 0; t + 1 < nl; ++t) {
        const SoloLevel& S = plan.solo[t];
        const CoarseLevel<T>& L = c.L[js + t];
        T* X = P_(S.o_x);
        T* Y = P_(S.o_y);
        const T* d = P_(S.o_dinv);
        const T* b = P_(S.o_b);
        for (int32_t i = threadIdx.x; i < S.n; i += blockDim.x) X[i] = (T)(L.sm_omega[0] * (double)d[i] * (double)b[i]);
        __syncthreads();
        T* cu = X;
        T* ot = Y;
        for (int s = 1; s < nu; ++s) {
            sweep(S, cu, s == 1 ? nullptr : ot, L.sm_omega[s], L.sm_alpha[s], ot);
            T* tt = cu; cu = ot; ot = tt;
        }
        curs[t] = cu;
        {   // t_i = P_i (b_i - (A x)_i)
            const T* Pv = P_(S.o_P);
            T* tv = P_(S.o_t);
            for (int32_t base = w.warp * RRPW; base < S.n; base += RWARPS * RRPW) {
                const int32_t i = base + w.sub;
                const bool valid = i < S.n;
                const double sum = rowsum(S, i, valid, cu);
                if (valid && w.sl == 0) tv[i] = (T)((double)Pv[i] * ((double)b[i] - sum));
            }
            __syncthreads();
        }
        {   // b_next[a] = sum over the members of a (ascending) of t
            const SoloLevel& N = plan.solo[t + 1];
            const int64_t* mp = reinterpret_cast<const int64_t*>(sm + S.o_mp);
            const int32_t* ml = reinterpret_cast<const int32_t*>(sm + S.o_ml);
            const T* tv = P_(S.o_t);
            T* bn = P_(N.o_b);
            for (int32_t base = w.warp * RRPW; base < N.n; base += RWARPS * RRPW) {
                const int32_t a = base + w.sub;
                double sum = 0.0;
                if (a < N.n)
                    for (int64_t e = mp[a] + w.sl; e < mp[a + 1]; e += RSVL) sum += (double)tv[ml[e]];
                sum = group_sum<RSVL>(sum);
                if (a < N.n && w.sl == 0) bn[a] = (T)sum;
            }
            __syncthreads();
        }
    }
    {   // coarsest: z = A_c^-1 b (fp64 rows)
        const SoloLevel& C = plan.solo[nl - 1];
        const double* Ai = reinterpret_cast<const double*>(sm + C.o_val);
        const T* bc = P_(C.o_b);
        T* zc = P_(C.o_z);
        for (int32_t i = w.warp; i < C.n; i += RWARPS) {
            double s = 0.0;
            for (int32_t j = w.lane; j < C.n; j += 32) s += Ai[(int64_t)i * C.n + j] * (double)bc[j];
            s = group_sum<32>(s);
            if (w.lane == 0) zc[i] = (T)s;
        }
        __syncthreads();
    }
    for (int t = nl - 2; t >= 0; --t) {
        const SoloLevel& S = plan.solo[t];
        const CoarseLevel<T>& L = c.L[js + t];
        T* cu = curs[t];
        T* ot = cu == P_(S.o_x) ? P_(S.o_y) : P_(S.o_x);
        const T* zc = P_(plan.solo[t + 1].o_z);
        const T* Pv = P_(S.o_P);
        const int32_t* agg = reinterpret_cast<const int32_t*>(sm + S.o_agg);
        for (int32_t i = threadIdx.x; i < S.n; i += blockDim.x)
            ot[i] = (T)((double)cu[i] + (double)Pv[i] * (double)zc[agg[i]]);
        __syncthreads();
        T* in = ot;
        T* out = cu;
        for (int s = 0; s < nu; ++s) {
            const bool last = s == nu - 1;
            T* dst = last ? (t == 0 ? c.L[js].z : P_(S.o_z)) : out;
            sweep(S, in, s == 0 ? nullptr : out, L.sm_omega[s], s == 0 ? 0.0 : L.sm_alpha[s], dst);
            if (!last) { T* tt = in; in = out; out = tt; }
        }
    }
}

template <class T>
__global__ void __launch_bounds__(RB, 1) k_coarse_vcycle_res(const __grid_constant__ CoarseCycle<T> c,
                                                             const __grid_constant__ ResPlan plan, int mode,
                                                             int kstop, const __grid_constant__ TailArgs<T> ta,
                                                             uint32_t tail_base) {
    // mode 0: the whole cycle; 1: down phase of levels 0..kstop-1 (ends with b of level kstop); 2: up phase
    // from level kstop-1 (z of level kstop given) — levels >= kstop then run on the cluster tail kernel;
    // 3: 1, then the tail on the first cluster of this (cooperative + cluster) launch, then 2 — one launch
    __shared__ TailLevel tail_lv[TAIL_MAXL];
    __shared__ __align__(8) uint64_t tail_bar;
    __shared__ __align__(8) uint64_t tail_pbars[2];
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar_late;
    __shared__ CoarseCycle<T> sc;
    __shared__ ResLevel slv[16];  // this CTA's slice descriptors (read after every barrier)
    const Lanes w;
    const int cta = blockIdx.x;
    if (c.trace && blockIdx.x == 0 && threadIdx.x == 0) {  // kernel entry (before the shared-memory staging)
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        c.trace[96 + (mode == 2 ? 2 : 0)] = t0;
    }
    {
        const int* src = reinterpret_cast<const int*>(&c);
        int* dst = reinterpret_cast<int*>(&sc);
        for (int k = threadIdx.x; k < (int)(sizeof(CoarseCycle<T>) / sizeof(int)); k += blockDim.x) dst[k] = src[k];
        const int* ls = reinterpret_cast<const int*>(plan.lv + (size_t)cta * 16);
        int* ld = reinterpret_cast<int*>(slv);
        for (int k = threadIdx.x; k < (int)(16 * sizeof(ResLevel) / sizeof(int)); k += blockDim.x) ld[k] = ls[k];
    }
    if (threadIdx.x == 0) {  // this CTA's slices of every level -> shared memory
        // two completion barriers: the first cycle level's slices (bar) and the rest (bar_late, flagged by the
        // plan in bit 31 of the byte count), so the first phases start before the deeper levels have landed
        mbar_init(&bar, 1);
        mbar_init(&bar_late, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const ResCopy* cp = plan.copies + (size_t)cta * RES_MAXC;
        uint32_t early = 0, late = 0;
        for (int k = 0; k < plan.ncopies[cta]; ++k) {
            const uint32_t by = cp[k].bytes & RES_BYTES_MASK;
            if (cp[k].bytes & RES_LATE) late += by;
            else early += by;
        }
        mbar_expect_tx(&bar, early);
        mbar_expect_tx(&bar_late, late);
        for (int k = 0; k < plan.ncopies[cta]; ++k)
            bulk_g2s(smem + cp[k].dst, cp[k].src, cp[k].bytes & RES_BYTES_MASK, (cp[k].bytes & RES_LATE) ? &bar_late : &bar);
    }
    __syncthreads();
    // mode 3: the first cluster also stages its static tail data now, behind the grid levels' work
    if (mode == 3 && blockIdx.x < (unsigned)ta.CT) tail_detail::coarse_tail_load<T>(ta, smem + tail_base, tail_lv, tail_bar, tail_pbars);
    mbar_wait(&bar, 0);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // (PDL launch: the previous kernel's b is complete)
    int tix = 0;
    auto mark = [&]() {
        if (c.trace && blockIdx.x == 0 && threadIdx.x == 0 && tix < 64) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            c.trace[tix] = t;
        }
        ++tix;
    };
    mark();
    const int K = sc.K, nu = sc.nu;
    auto slice = [&](int k) { return Slice<T>{smem, slv[k]}; };
    T* cur[16];
    const bool solo_on = mode == 0 && plan.solo[0].n > 0;   // cycle levels solo..K-1 on CTA 0 alone
    const int solo = solo_on ? plan.solo_first : 0;
    const int kdown = mode == 0 ? (solo_on ? solo : K - 1) : kstop;
    bool late_ready = false;
    auto wait_late = [&]() {
        if (!late_ready) { mbar_wait(&bar_late, 0); late_ready = true; }
    };
    if (mode == 2) wait_late();
    // ---- down
    for (int k = 0; k < kdown && mode != 2; ++k) {
        if (k == 1) wait_late();
        const CoarseLevel<T>& L = sc.L[k];
        const Slice<T> S = slice(k);
        const T* __restrict__ b = L.b;
        const T* __restrict__ d = L.dinv;
        const double om0 = L.sm_omega[0];
        auto x1f = [&](int32_t j) { return (T)(om0 * (double)d[j] * (double)b[j]); };
        auto zero = [&](int32_t) { return (T)0; };
        T* cu = L.x;
        T* ot = L.y;
        if (nu >= 2) {
            sweep(w, L, S, x1f, zero, L.sm_omega[1], L.sm_alpha[1], L.x);
            for (int s = 2; s < nu; ++s) {
                grid.sync(); mark();
                const T* __restrict__ src = cu;
                T* __restrict__ prv = ot;
                if (s == 2) sweep(w, L, S, [&](int32_t j) { return src[j]; }, x1f, L.sm_omega[s], L.sm_alpha[s], ot);
                else sweep(w, L, S, [&](int32_t j) { return src[j]; }, [&](int32_t i) { return prv[i]; },
                           L.sm_omega[s], L.sm_alpha[s], ot);
                T* t = cu; cu = ot; ot = t;
            }
        } else {
            for (int64_t i = S.d.r0 + threadIdx.x; i < S.d.r1; i += blockDim.x) L.x[i] = x1f((int32_t)i);
        }
        cur[k] = cu;
        grid.sync(); mark();
        resid(w, L, S, cu);
        grid.sync(); mark();
        restrict_t(w, L, S, sc.L[k + 1].b);
        grid.sync(); mark();
    }
    if (mode == 1) return;
    wait_late();
    if (solo_on) {  // the smallest levels on CTA 0, whole in its shared memory, __syncthreads between phases
        if (blockIdx.x == 0) solo_cycle<T>(w, sc, plan, solo, smem);
        grid.sync(); mark();
    }
    if (mode == 3) {  // the tail levels on the first cluster while the other CTAs wait at the grid barrier
        if (blockIdx.x < (unsigned)ta.CT) tail_detail::coarse_tail_body<T>(ta, smem + tail_base, tail_lv, tail_bar, tail_pbars);
        grid.sync(); mark();
    }
    // ---- coarsest
    if (mode == 0 && !solo_on) dense_solve(w, sc.L[K - 1].n, slice(K - 1), sc.L[K - 1].b, sc.L[K - 1].z);
    // ---- up
    for (int k = mode == 0 ? (solo_on ? solo - 1 : K - 2) : kstop - 1; k >= 0; --k) {
        const CoarseLevel<T>& L = sc.L[k];
        const Slice<T> S = slice(k);
        // the buffer the down phase left the pre-smoothed x in (mode 2: recomputed from nu)
        T* __restrict__ cu = mode == 2 ? ((nu >= 2 && ((nu - 2) & 1)) ? L.y : L.x) : cur[k];
        T* ot = cu == L.x ? L.y : L.x;
        const T* __restrict__ zc = sc.L[k + 1].z;
        const T* __restrict__ P = L.P;
        const int32_t* __restrict__ agg = L.agg;
        const bool mat = L.n >= 32768;
        auto zero = [&](int32_t) { return (T)0; };
        grid.sync(); mark();
        if (mat) {  // materialise x_0 = x + P z_c[agg] over the owned rows (shared-memory P, agg)
            for (int64_t i = S.d.r0 + threadIdx.x; i < S.d.r1; i += blockDim.x)
                cu[i] = (T)((double)cu[i] + (double)S.P(i) * (double)zc[S.agg(i)]);
            grid.sync(); mark();
        }
        auto x0f = [&](int32_t j) { return mat ? cu[j] : (T)((double)cu[j] + (double)P[j] * (double)zc[agg[j]]); };
        T* src = nu == 1 ? L.z : ot;
        sweep(w, L, S, x0f, zero, L.sm_omega[0], 0.0, src);
        T* prv = cu;
        for (int s = 1; s < nu; ++s) {
            grid.sync(); mark();
            T* out = s == nu - 1 ? L.z : prv;
            const T* __restrict__ xs = src;
            const T* __restrict__ xp = prv;
            if (s == 1) sweep(w, L, S, [&](int32_t j) { return xs[j]; }, x0f, L.sm_omega[s], L.sm_alpha[s], out);
            else sweep(w, L, S, [&](int32_t j) { return xs[j]; }, [&](int32_t i) { return xp[i]; }, L.sm_omega[s],
                       L.sm_alpha[s], out);
            prv = src;
            src = out;
        }
    }
}

}  // namespace

template <class T>
bool coarse_res_plan(const CoarseCycle<T>& c, int G, uint32_t smem_cap, std::vector<ResLevel>& lv,
                     std::vector<ResCopy>& copies, std::vector<int32_t>& ncopies, std::vector<uint32_t>& tx,
                     uint32_t& smem, cudaStream_t s, bool with_coarsest, ResPlan* solo_out) {
    const int K = c.K;
    if (K < 2 || K > 16) return false;
    std::vector<std::vector<int32_t>> rb(K), ab(K);
    std::vector<std::vector<int64_t>> rp(K), mp(K);
    for (int k = 0; k < K; ++k) {
        const CoarseLevel<T>& L = c.L[k];
        if (k + 1 < K) {
            rp[k].resize((size_t)L.n + 1);
            d2h(rp[k].data(), L.rowptr, (size_t)L.n + 1, s);
            mp[k].resize((size_t)L.n_agg + 1);
            d2h(mp[k].data(), L.mptr, (size_t)L.n_agg + 1, s);
        }
    }
    MG_CK(cudaStreamSynchronize(s));
    for (int k = 0; k < K; ++k) {
        const CoarseLevel<T>& L = c.L[k];
        if (k + 1 < K) {
            rb[k] = partition_rows(rp[k].data(), L.n, G);             // rows balanced by nonzeros
            ab[k] = partition_rows(mp[k].data(), L.n_agg, G);         // aggregates balanced by members
        } else {
            rb[k].resize(G + 1);
            for (int g = 0; g <= G; ++g) rb[k][g] = (int32_t)((int64_t)L.n * g / G);
        }
    }
    lv.assign((size_t)G * 16, ResLevel());
    copies.assign((size_t)G * RES_MAXC, ResCopy{nullptr, 0, 0});
    ncopies.assign(G, 0);
    tx.assign(G, 0);
    smem = 0;
    for (int g = 0; g < G; ++g) {
        uint32_t cursor = 0;
        int nc = 0;
        bool late_lv = false;  // copies of cycle levels >= 1 (and the solo tail) complete on the kernel's second barrier
        auto add = [&](uint32_t& off, const void* base, int64_t elem_off, size_t esz, size_t count) -> bool {
            const uintptr_t src = reinterpret_cast<uintptr_t>(base) + (uintptr_t)(elem_off * (int64_t)esz);
            const uintptr_t al = src & ~(uintptr_t)15;
            const uint32_t lead = (uint32_t)(src - al);
            const uint32_t dst = (cursor + 15u) & ~15u;
            off = dst + lead;
            const size_t bytes = count * esz;
            if (bytes == 0) { cursor = dst; return true; }
            const uint32_t nb = (uint32_t)((lead + bytes + 15) & ~(size_t)15);
            if (nc >= RES_MAXC) return false;
            copies[(size_t)g * RES_MAXC + nc++] = ResCopy{reinterpret_cast<const void*>(al), dst, nb | (late_lv ? RES_LATE : 0u)};
            cursor = dst + nb;
            tx[g] += nb;
            return true;
        };
        for (int k = 0; k < K; ++k) {
            late_lv = k > 0;
            const CoarseLevel<T>& L = c.L[k];
            ResLevel& d = lv[(size_t)g * 16 + k];
            d.r0 = rb[k][g]; d.r1 = rb[k][g + 1];
            const int64_t rows = d.r1 - d.r0;
            bool ok = true;
            if (k + 1 < K) {
                d.e0 = rp[k][d.r0];
                const int64_t nnz = rp[k][d.r1] - d.e0;
                d.a0 = ab[k][g]; d.a1 = ab[k][g + 1];
                d.m0 = mp[k][d.a0];
                const int64_t mem = mp[k][d.a1] - d.m0;
                ok = ok && add(d.o_rp, L.rowptr, d.r0, 8, (size_t)rows + 1);
                ok = ok && add(d.o_col, L.col, d.e0, 4, (size_t)nnz);
                ok = ok && add(d.o_val, L.val, d.e0, sizeof(T), (size_t)nnz);
                ok = ok && add(d.o_dinv, L.dinv, d.r0, sizeof(T), (size_t)rows);
                ok = ok && add(d.o_P, L.P, d.r0, sizeof(T), (size_t)rows);
                ok = ok && add(d.o_agg, L.agg, d.r0, 4, (size_t)rows);
                ok = ok && add(d.o_mp, L.mptr, d.a0, 8, (size_t)(d.a1 - d.a0) + 1);
                ok = ok && add(d.o_ml, L.mlist, d.m0, 4, (size_t)mem);
            } else if (with_coarsest) {
                ok = ok && add(d.o_val, c.Ainv, (int64_t)d.r0 * L.n, 8, (size_t)rows * L.n);
            }
            if (!ok) return false;
        }
        late_lv = true;
        if (g == 0 && solo_out && with_coarsest) {   // the solo tail in CTA 0 (coarse_res.cuh)
            const size_t ts = sizeof(T);
            auto level_bytes = [&](int k) -> size_t {
                const CoarseLevel<T>& L = c.L[k];
                if (k + 1 == K) return (size_t)L.n * L.n * 8 + 2 * (size_t)L.n * ts + 64;
                const size_t nnz = (size_t)rp[k][L.n];
                return ((size_t)L.n + 1) * 8 + nnz * (4 + ts) + (size_t)L.n * (2 * ts + 8) + ((size_t)L.n_agg + 1) * 8 +
                       5 * (size_t)L.n * ts + 16 * 16;
            };
            int js = K;
            size_t tot = 0;
            for (int k = K - 1; k >= 0; --k) {
                if (k + 1 < K && c.L[k].n > 8192) break;
                if (cursor + tot + level_bytes(k) > smem_cap || K - k > SOLO_MAXL) break;
                tot += level_bytes(k);
                js = k;
            }
            solo_out->solo_first = 0;
            if (js <= K - 2) {
                uint32_t save_cursor = cursor;
                int save_nc = nc;
                uint32_t save_tx = tx[g];
                bool ok = true;
                for (int k = js; k < K && ok; ++k) {
                    const CoarseLevel<T>& L = c.L[k];
                    SoloLevel& d = solo_out->solo[k - js];
                    d = SoloLevel();
                    d.n = L.n;
                    auto vec = [&](uint32_t& off) { off = (cursor + 15u) & ~15u; cursor = off + (uint32_t)((size_t)L.n * ts); };
                    if (k + 1 < K) {
                        const int64_t nnz = rp[k][L.n];
                        ok = ok && add(d.o_rp, L.rowptr, 0, 8, (size_t)L.n + 1);
                        ok = ok && add(d.o_col, L.col, 0, 4, (size_t)nnz);
                        ok = ok && add(d.o_val, L.val, 0, ts, (size_t)nnz);
                        ok = ok && add(d.o_dinv, L.dinv, 0, ts, (size_t)L.n);
                        ok = ok && add(d.o_P, L.P, 0, ts, (size_t)L.n);
                        ok = ok && add(d.o_agg, L.agg, 0, 4, (size_t)L.n);
                        ok = ok && add(d.o_mp, L.mptr, 0, 8, (size_t)L.n_agg + 1);
                        ok = ok && add(d.o_ml, L.mlist, 0, 4, (size_t)L.n);
                        vec(d.o_x); vec(d.o_y); vec(d.o_t);
                    } else {
                        ok = ok && add(d.o_val, c.Ainv, 0, 8, (size_t)L.n * L.n);
                    }
                    vec(d.o_b); vec(d.o_z);
                }
                if (ok && cursor <= smem_cap) {
                    solo_out->solo_first = js;
                } else {
                    cursor = save_cursor; nc = save_nc; tx[g] = save_tx;
                }
            }
        }
        ncopies[g] = nc;
        smem = std::max(smem, cursor);
        if (cursor > smem_cap) return false;
    }
    return true;
}

template <class T>
void coarse_vcycle_res(const CoarseCycle<T>& c, const ResPlan& plan, cudaStream_t s, int mode, int kstop,
                       const TailArgs<T>* tail, uint32_t tail_base, uint32_t tail_smem) {
    const uint32_t smem = mode == 3 ? tail_base + tail_smem : plan.smem;
    ensure_dyn_smem((const void*)k_coarse_vcycle_res<T>, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.G);
    cfg.blockDim = dim3(RB);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr_[3];
    attr_[0].id = cudaLaunchAttributeCooperative;
    attr_[0].val.cooperative = 1;
    int na = 1;
    if (mode == 3) {
        attr_[na].id = cudaLaunchAttributeClusterDimension;
        attr_[na].val.clusterDim.x = (unsigned)tail->CT;
        attr_[na].val.clusterDim.y = 1; attr_[na].val.clusterDim.z = 1;
        ++na;
    }
    // programmatic dependent launch (MGPBD_COARSE_PDL): the CTAs stage their static slices while the preceding
    // kernel (the level-0 restriction) finishes; griddepcontrol.wait precedes the first read of b
    const bool pdl = std::getenv("MGPBD_COARSE_PDL") != nullptr;
    if (pdl && (mode == 0 || mode == 1 || mode == 3)) {
        attr_[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr_[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr_;
    cfg.numAttrs = na;
    TailArgs<T> ta;
    if (tail) ta = *tail;
    MG_CK(cudaLaunchKernelEx(&cfg, k_coarse_vcycle_res<T>, c, plan, mode, kstop, ta, tail_base));
    MG_LAUNCH_CHECK();
}

// Co-resident CTAs of a cooperative launch of the fused (mode 3) kernel in clusters of CT with `smem` bytes
// (a multiple of CT; 0: not launchable).
template <class T>
int coarse_res_fused_grid(int CT, uint32_t smem) {
    if (!try_raise_dyn_smem((const void*)k_coarse_vcycle_res<T>, smem)) return 0;
    if (CT > 8 && cudaFuncSetAttribute((const void*)k_coarse_vcycle_res<T>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                       1) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CT);
    cfg.blockDim = dim3(RB);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CT; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (const void*)k_coarse_vcycle_res<T>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return nc * CT;
}

template <class T>
int coarse_res_blocks_per_sm(uint32_t smem) {
    if (!try_raise_dyn_smem((const void*)k_coarse_vcycle_res<T>, smem)) return 0;  // raise-only (util.cu)
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_coarse_vcycle_res<T>, RB, smem) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return nb;
}

#define MG_INST(T)                                                                                             \
    template bool coarse_res_plan<T>(const CoarseCycle<T>&, int, uint32_t, std::vector<ResLevel>&,             \
                                     std::vector<ResCopy>&, std::vector<int32_t>&, std::vector<uint32_t>&,     \
                                     uint32_t&, cudaStream_t, bool, ResPlan*);                                 \
    template void coarse_vcycle_res<T>(const CoarseCycle<T>&, const ResPlan&, cudaStream_t, int, int,         \
                                       const TailArgs<T>*, uint32_t, uint32_t);                                \
    template int coarse_res_fused_grid<T>(int, uint32_t);                                                      \
    template int coarse_res_blocks_per_sm<T>(uint32_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
