// Persistent cooperative coarse V-cycle, see coarse.cuh.
//
// Every phase is latency-bound: after a grid barrier a lane group's critical path is the chain of
// dependent global loads (rowptr -> col/val -> x).  The matrix, prolongator and aggregate lists do
// not change during a cycle, so each lane group loads the static part of its FIRST row (or aggregate)
// of the next phase before it waits at the barrier; after the barrier only the vector gathers remain.
// (Level 1 needs a few row waves; the smaller levels fit in one.)
#include <cooperative_groups.h>

#include <algorithm>

#include "coarse.cuh"

namespace cg = cooperative_groups;

namespace mgpbd {

namespace {

constexpr int CB = 512;   // threads per CTA
constexpr int SVL = 8;    // lanes per row
constexpr int SCH = 5;    // nonzeros per lane per chunk (all loads of a chunk issued before use)
constexpr int RPW = 32 / SVL;
constexpr int CHUNK = SVL * SCH;

struct Lanes {
    int lane, sub, sl;
    int64_t gw, nw;  // global warp index, warps in the grid
    __device__ Lanes() {
        lane = threadIdx.x & 31;
        sub = lane / SVL;
        sl = lane % SVL;
        gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    }
};

// static part of one row for this lane: range and the first chunk of (col, val)
template <class T>
struct Pre {
    int64_t a, e;
    int32_t c[SCH];
    T v[SCH];
};

template <class T>
__device__ __forceinline__ void pre_row(const Lanes& w, const CoarseLevel<T>& L, bool valid, int64_t i, Pre<T>& p) {
    p.a = valid ? L.rowptr[i] : 0;
    p.e = valid ? L.rowptr[i + 1] : 0;
#pragma unroll
    for (int q = 0; q < SCH; ++q) {
        const int64_t k = p.a + q * SVL + w.sl;
        const bool in = k < p.e;
        p.c[q] = in ? L.col[k] : -1;
        p.v[q] = in ? L.val[k] : (T)0;
    }
}

// sum_k A_ik x(col_k) for the lane group's row; chunk 0 from the prefetched p, later chunks loaded
// here (the loop runs to the warp's longest row so the butterfly sees the whole warp).  Products and
// lane partials in T, butterfly in T, result in fp64 (the per-level kernels' precision).
template <class T, class XF>
__device__ __forceinline__ double row_sum(const Lanes& w, const CoarseLevel<T>& L, const Pre<T>& p, XF xf) {
    const int maxlen = __reduce_max_sync(0xffffffffu, (int)(p.e - p.a));
    T xv[SCH];
#pragma unroll
    for (int q = 0; q < SCH; ++q) xv[q] = p.c[q] >= 0 ? xf(p.c[q]) : (T)0;
    T part = (T)0;
#pragma unroll
    for (int q = 0; q < SCH; ++q) part += p.v[q] * xv[q];
    for (int off = CHUNK; off < maxlen; off += CHUNK) {
        int32_t c[SCH];
        T v[SCH];
#pragma unroll
        for (int q = 0; q < SCH; ++q) {
            const int64_t k = p.a + off + q * SVL + w.sl;
            const bool in = k < p.e;
            c[q] = in ? L.col[k] : -1;
            v[q] = in ? L.val[k] : (T)0;
        }
#pragma unroll
        for (int q = 0; q < SCH; ++q) xv[q] = c[q] >= 0 ? xf(c[q]) : (T)0;
#pragma unroll
        for (int q = 0; q < SCH; ++q) part += v[q] * xv[q];
    }
    return (double)group_sum_t<SVL>(part);
}

// row-parallel phases: lane group `sub` of warp gw handles rows gw*RPW + sub + t*nw*RPW
template <class T>
__device__ __forceinline__ void pre_rows(const Lanes& w, const CoarseLevel<T>& L, Pre<T>& p) {
    const int64_t i = w.gw * RPW + w.sub;
    pre_row(w, L, i < L.n, i, p);
}

// One smoother step over all rows: y = x + alpha (x - xprev) + omega D^-1 (b - A x), x given by xf(j)
// (materialised vector or an on-the-fly expression), xprev by xpf(i) (row-local; unused if alpha = 0).
template <class T, class XF, class XPF>
__device__ __forceinline__ void sweep(const Lanes& w, const CoarseLevel<T>& L, Pre<T>& p, XF xf, XPF xpf, double omega,
                                      double alpha, T* __restrict__ out) {
    for (int64_t base = w.gw * RPW; base < L.n; base += w.nw * RPW) {  // warp-uniform trip count
        const int64_t i = base + w.sub;
        const bool valid = i < L.n;
        if (base != w.gw * RPW) pre_row(w, L, valid, i, p);
        const double s = row_sum(w, L, p, xf);
        if (valid && w.sl == 0) {
            const double xi = (double)xf((int32_t)i);
            double y = xi + omega * (double)L.dinv[i] * ((double)L.b[i] - s);
            if (alpha != 0.0) y += alpha * (xi - (double)xpf((int32_t)i));
            out[i] = (T)y;
        }
    }
}

// t_i = P_i (b_i - (A x)_i) for all rows (row-parallel half of the residual/restriction)
template <class T>
__device__ __forceinline__ void resid(const Lanes& w, const CoarseLevel<T>& L, Pre<T>& p, const T* __restrict__ x) {
    for (int64_t base = w.gw * RPW; base < L.n; base += w.nw * RPW) {
        const int64_t i = base + w.sub;
        const bool valid = i < L.n;
        if (base != w.gw * RPW) pre_row(w, L, valid, i, p);
        const double s = row_sum(w, L, p, [&](int32_t j) { return x[j]; });
        if (valid && w.sl == 0) L.t[i] = (T)((double)L.P[i] * ((double)L.b[i] - s));
    }
}

// restriction: SVL lanes per aggregate; static part = member range and the first member per lane
struct PreAgg {
    int64_t m0, m1;
    int32_t i;
};
template <class T>
__device__ __forceinline__ void pre_agg(const Lanes& w, const CoarseLevel<T>& L, int64_t a, PreAgg& q) {
    const bool valid = a < L.n_agg;
    q.m0 = valid ? L.mptr[a] : 0;
    q.m1 = valid ? L.mptr[a + 1] : 0;
    q.i = q.m0 + w.sl < q.m1 ? L.mlist[q.m0 + w.sl] : -1;
}

// bnext[a] = sum_{i in a, ascending} t_i: lane-strided members + fixed butterfly
template <class T>
__device__ __forceinline__ void restrict_t(const Lanes& w, const CoarseLevel<T>& L, PreAgg& q, T* __restrict__ bnext) {
    for (int64_t base = w.gw * RPW; base < L.n_agg; base += w.nw * RPW) {  // warp-uniform trip count
        const int64_t a = base + w.sub;
        if (base != w.gw * RPW) pre_agg(w, L, a, q);
        double s = q.i >= 0 ? (double)L.t[q.i] : 0.0;
        for (int64_t e = q.m0 + w.sl + SVL; e < q.m1; e += SVL) s += (double)L.t[L.mlist[e]];
        s = group_sum<SVL>(s);
        if (a < L.n_agg && w.sl == 0) bnext[a] = (T)s;
    }
}

// fused residual + restriction for small levels: one warp per aggregate, RPW member rows at a time
// (members in ascending order); static part = the first batch's member rows
template <class T>
struct PreFused {
    int64_t m0, m1;
    int32_t i;
    Pre<T> r;
};
template <class T>
__device__ __forceinline__ void pre_fused(const Lanes& w, const CoarseLevel<T>& L, int64_t a, PreFused<T>& f) {
    const bool va = a < L.n_agg;
    f.m0 = va ? L.mptr[a] : 0;
    f.m1 = va ? L.mptr[a + 1] : 0;
    const bool valid = f.m0 + w.sub < f.m1;
    f.i = valid ? L.mlist[f.m0 + w.sub] : 0;
    pre_row(w, L, valid, f.i, f.r);
}

template <class T>
__device__ __forceinline__ void resid_restrict(const Lanes& w, const CoarseLevel<T>& L, PreFused<T>& f,
                                               const T* __restrict__ x, T* __restrict__ bnext) {
    for (int64_t a = w.gw; a < L.n_agg; a += w.nw) {
        if (a != w.gw) pre_fused(w, L, a, f);
        double acc = 0.0;
        for (int64_t mb = f.m0; mb < f.m1; mb += RPW) {
            const bool valid = mb + w.sub < f.m1;
            int32_t i = f.i;
            if (mb != f.m0) {
                i = valid ? L.mlist[mb + w.sub] : 0;
                pre_row(w, L, valid, i, f.r);
            }
            const double s = row_sum(w, L, f.r, [&](int32_t j) { return x[j]; });
            const double t = valid ? (double)(T)((double)L.P[i] * ((double)L.b[i] - s)) : 0.0;
#pragma unroll
            for (int g = 0; g < RPW; ++g) acc += __shfl_sync(0xffffffffu, t, g * SVL);
        }
        if (w.lane == 0) bnext[a] = (T)acc;
    }
}

template <class T>
__device__ __forceinline__ void dense_solve(const Lanes& w, int32_t n, const double* __restrict__ Ainv,
                                            const T* __restrict__ b, T* __restrict__ x) {
    for (int64_t i = w.gw; i < n; i += w.nw) {
        double s = 0.0;
        for (int32_t j = w.lane; j < n; j += 32) s += Ainv[i * n + j] * (double)b[j];
        s = group_sum<32>(s);
        if (w.lane == 0) x[i] = (T)s;
    }
}

template <class T>
__device__ __forceinline__ bool fused_level(const CoarseLevel<T>& L) {
    return L.n_agg < 500;  // small level: one phase (warp per aggregate) beats two
}

template <class T>
__global__ void __launch_bounds__(CB, 2) k_coarse_vcycle(const __grid_constant__ CoarseCycle<T> c) {
    cg::grid_group grid = cg::this_grid();
    const Lanes w;
    // the cycle descriptor in shared memory: level fields are read after every barrier
    __shared__ CoarseCycle<T> sc;
    {
        const int* src = reinterpret_cast<const int*>(&c);
        int* dst = reinterpret_cast<int*>(&sc);
        for (int k = threadIdx.x; k < (int)(sizeof(CoarseCycle<T>) / sizeof(int)); k += blockDim.x) dst[k] = src[k];
        __syncthreads();
    }
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
    T* cur[16];
    Pre<T> p;
    PreAgg q;
    PreFused<T> f;
    // ---- down
    if (K > 1) pre_rows(w, sc.L[0], p);
    for (int k = 0; k + 1 < K; ++k) {
        const CoarseLevel<T>& L = sc.L[k];
        const T* __restrict__ b = L.b;
        const T* __restrict__ d = L.dinv;
        const double om0 = L.sm_omega[0];
        auto x1f = [&](int32_t j) { return (T)(om0 * (double)d[j] * (double)b[j]); };  // step 0 from x = 0
        auto zero = [&](int32_t) { return (T)0; };
        T* cu = L.x;
        T* ot = L.y;
        if (nu >= 2) {
            // pre-smoothing: step 0 (x_1 = omega_0 D^-1 b) evaluated on the fly inside step 1 (x_0 = 0)
            sweep(w, L, p, x1f, zero, L.sm_omega[1], L.sm_alpha[1], L.x);
            for (int s = 2; s < nu; ++s) {  // step s: x_{s+1} written over x_{s-1} (row-local read first)
                pre_rows(w, L, p);
                grid.sync(); mark();
                const T* __restrict__ src = cu;
                T* __restrict__ prv = ot;
                if (s == 2) sweep(w, L, p, [&](int32_t j) { return src[j]; }, x1f, L.sm_omega[s], L.sm_alpha[s], ot);
                else sweep(w, L, p, [&](int32_t j) { return src[j]; }, [&](int32_t i) { return prv[i]; },
                           L.sm_omega[s], L.sm_alpha[s], ot);
                T* t = cu; cu = ot; ot = t;
            }
        } else {
            for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += (int64_t)gridDim.x * blockDim.x)
                L.x[i] = x1f((int32_t)i);
        }
        cur[k] = cu;
        if (fused_level(L)) {
            pre_fused(w, L, w.gw, f);
            grid.sync(); mark();
            resid_restrict(w, L, f, cu, sc.L[k + 1].b);
        } else {  // row-parallel residual, then restriction
            pre_rows(w, L, p);
            grid.sync(); mark();
            resid(w, L, p, cu);
            pre_agg(w, L, w.gw * RPW + w.sub, q);
            grid.sync(); mark();
            restrict_t(w, L, q, sc.L[k + 1].b);
        }
        if (k + 2 < K) pre_rows(w, sc.L[k + 1], p);
        grid.sync(); mark();
    }
    // ---- coarsest
    dense_solve(w, sc.L[K - 1].n, sc.Ainv, sc.L[K - 1].b, sc.L[K - 1].z);
    // ---- up
    for (int k = K - 2; k >= 0; --k) {
        const CoarseLevel<T>& L = sc.L[k];
        T* __restrict__ cu = cur[k];
        T* ot = cu == L.x ? L.y : L.x;
        const T* __restrict__ zc = sc.L[k + 1].z;
        const T* __restrict__ P = L.P;
        const int32_t* __restrict__ agg = L.agg;
        const bool mat = L.n >= 32768;
        auto zero = [&](int32_t) { return (T)0; };
        if (mat) {
            // large level: materialise x_0 = x + P z_c[agg] (row-local; static operands loaded before
            // the barrier) — cheaper than three extra gathers per nonzero in the next step
            const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
            const int64_t nt = (int64_t)gridDim.x * blockDim.x;
            int32_t a0 = 0;
            double x0 = 0.0, p0 = 0.0;
            if (tid < L.n) { a0 = agg[tid]; x0 = (double)cu[tid]; p0 = (double)P[tid]; }
            grid.sync(); mark();
            for (int64_t i = tid; i < L.n; i += nt) {
                if (i != tid) { a0 = agg[i]; x0 = (double)cu[i]; p0 = (double)P[i]; }
                cu[i] = (T)(x0 + p0 * (double)zc[a0]);
            }
        }
        // x_0 of the post-smoothing: materialised, or the prolongation evaluated on the fly
        auto x0f = [&](int32_t j) { return mat ? cu[j] : (T)((double)cu[j] + (double)P[j] * (double)zc[agg[j]]); };
        pre_rows(w, L, p);
        grid.sync(); mark();
        T* src = nu == 1 ? L.z : ot;
        sweep(w, L, p, x0f, zero, L.sm_omega[0], 0.0, src);  // step 0 (alpha_0 = 0)
        T* prv = cu;                                          // buffer of x_{s-1}
        for (int s = 1; s < nu; ++s) {
            pre_rows(w, L, p);
            grid.sync(); mark();
            T* out = s == nu - 1 ? L.z : prv;                  // over x_{s-1} (row-local read first)
            const T* __restrict__ xs = src;
            const T* __restrict__ xp = prv;
            if (s == 1) sweep(w, L, p, [&](int32_t j) { return xs[j]; }, x0f, L.sm_omega[s], L.sm_alpha[s], out);
            else sweep(w, L, p, [&](int32_t j) { return xs[j]; }, [&](int32_t i) { return xp[i]; }, L.sm_omega[s],
                       L.sm_alpha[s], out);
            prv = src;
            src = out;
        }
    }
}

template <class T>
int coarse_grid() {
    static const int g = [] {  // thread-safe one-time initialisation
        int dev = 0, sms = 0, occ = 0;
        MG_CK(cudaGetDevice(&dev));
        MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coarse_vcycle<T>, CB, 0));
        if (occ < 1) throw Error(-1, "coarse_vcycle: kernel does not fit on an SM");
        return sms * std::min(occ, 4);
    }();
    return g;
}

}  // namespace

template <class T>
void coarse_vcycle(const CoarseCycle<T>& c, cudaStream_t s) {
    if (c.K < 1) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(coarse_grid<T>());
    cfg.blockDim = dim3(CB);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MG_CK(cudaLaunchKernelEx(&cfg, k_coarse_vcycle<T>, c));
    MG_LAUNCH_CHECK();
}

template void coarse_vcycle<float>(const CoarseCycle<float>&, cudaStream_t);
template void coarse_vcycle<double>(const CoarseCycle<double>&, cudaStream_t);

}  // namespace mgpbd
