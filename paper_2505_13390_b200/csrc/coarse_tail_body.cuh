// Device code of the cluster tail (coarse_tail.cuh), shared by the stand-alone tail kernel and the fused
// grid + cluster coarse kernel (coarse_res.cu).  Include only from .cu files.
#pragma once
#include <cooperative_groups.h>

#include "coarse_tail.cuh"
#include "tma.cuh"

namespace mgpbd {
namespace tail_detail {
namespace cg = cooperative_groups;

constexpr int TB = 1024;        // threads per CTA
constexpr int TVL = 8;          // lanes per row
constexpr int TCH = 5;          // nonzeros per lane per chunk
constexpr int TRPW = 32 / TVL;  // rows per warp
constexpr int TWARPS = TB / 32;

template <class U>
__device__ __forceinline__ U* sp(unsigned char* sm, uint32_t off) { return reinterpret_cast<U*>(sm + off); }

template <class T>
struct Tail {
    unsigned char* sm;
    cg::cluster_group cl;
    int CT, me;
    int lane, sub, sl, warp;

    // store value v at element `idx` of the buffer at smem offset `off` in every CTA of the cluster
    // (the 8 lanes of a row group share the CT stores)
    __device__ __forceinline__ void bcast_row(uint32_t off, int32_t idx, T v) {
        T* loc = sp<T>(sm, off) + idx;
        for (int r = sl; r < CT; r += TVL) *cl.map_shared_rank(loc, r) = v;
    }
    __device__ __forceinline__ void bcast_elem(uint32_t off, int32_t idx, T v, int r) {
        *cl.map_shared_rank(sp<T>(sm, off) + idx, r) = v;
    }

    // bulk mode: phases store their own rows locally (put), then publish() copies the own range to every other
    // CTA with one cp.async.bulk each (completion on the receiver's mbarrier; two barriers alternate so a fast
    // CTA's next broadcast can never complete a slower CTA's current phase) and waits for the others' ranges
    int bulk = 0, ph = 0;
    uint64_t* pbars = nullptr;
    __device__ __forceinline__ void put(uint32_t off, int32_t idx, T v) {
        if (bulk) { if (sl == 0) sp<T>(sm, off)[idx] = v; }
        else bcast_row(off, idx, v);
    }
    __device__ __forceinline__ void publish(const TailLevel& D, uint32_t off) {
        __syncthreads();
        uint64_t* bar = &pbars[ph & 1];
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, D.rx);
            const uint32_t src = smem_u32(sm + off + (size_t)D.r0 * sizeof(T));
            const uint32_t lbar = smem_u32(bar);
            if (D.ob)
                for (int r = 0; r < CT; ++r) {
                    if (r == me) continue;
                    uint32_t dst, rbar;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(src), "r"(r));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(lbar), "r"(r));
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                        "r"(src), "r"(D.ob), "r"(rbar)
                        : "memory");
                }
        }
        mbar_wait(bar, (uint32_t)((ph >> 1) & 1));
        ++ph;
    }

    // sum_k A_ik x[col_k] for own row i of level D (matrix and x in local shared memory)
    __device__ __forceinline__ double row_sum(const TailLevel& D, bool valid, int32_t i, uint32_t xoff) const {
        const int64_t* rp = sp<int64_t>(sm, D.o_rp);
        const uint16_t* col = sp<uint16_t>(sm, D.o_col);
        const T* val = sp<T>(sm, D.o_val);
        const T* x = sp<T>(sm, xoff);
        const int64_t a = valid ? rp[i - D.r0] - D.e0 : 0, e = valid ? rp[i - D.r0 + 1] - D.e0 : 0;
        const int maxlen = __reduce_max_sync(0xffffffffu, (int)(e - a));
        T part = (T)0;
        for (int off = 0; off < maxlen; off += TVL * TCH) {
            T v[TCH], xv[TCH];
#pragma unroll
            for (int q = 0; q < TCH; ++q) {
                const int64_t k = a + off + q * TVL + sl;
                const bool in = k < e;
                v[q] = in ? val[k] : (T)0;
                xv[q] = in ? x[col[k]] : (T)0;
            }
#pragma unroll
            for (int q = 0; q < TCH; ++q) part += v[q] * xv[q];
        }
        return (double)group_sum_t<TVL>(part);
    }
};

// The whole tail cycle on the calling cluster: smem = this CTA's tail region (identical offset in every CTA
// of the cluster), L / bar = a TailLevel[TAIL_MAXL] array and an mbarrier in static shared memory.
// Stage 1 (may run early: everything it copies is static for the cycle): this CTA's descriptors -> L, the
// bulk copies of its static tail data -> smem on `bar`; the two broadcast barriers pbars are initialised.
template <class T>
__device__ __forceinline__ void coarse_tail_load(const TailArgs<T>& A, unsigned char* smem, TailLevel* L, uint64_t& bar,
                                                 uint64_t* pbars) {
    const int me = (int)cg::this_cluster().block_rank();
    {
        const int* src = reinterpret_cast<const int*>(A.lv + (size_t)me * TAIL_MAXL);
        int* dst = reinterpret_cast<int*>(L);
        for (int k = threadIdx.x; k < (int)(TAIL_MAXL * sizeof(TailLevel) / sizeof(int)); k += TB) dst[k] = src[k];
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&pbars[0], 1);
        mbar_init(&pbars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&bar, A.txbytes[me]);
        const TailCopy* cp = A.copies + (size_t)me * TAIL_MAXC;
        for (int k = 0; k < A.ncopies[me]; ++k) bulk_g2s(smem + cp[k].dst, cp[k].src, cp[k].bytes, &bar);
    }
    __syncthreads();
}

// Stage 2: wait for stage 1, read the first tail level's rhs (own rows; written by whoever restricted into it)
// and run the cycle.
template <class T>
__device__ __forceinline__ void coarse_tail_body(const TailArgs<T>& A, unsigned char* smem, TailLevel* L, uint64_t& bar,
                                                 uint64_t* pbars) {
    Tail<T> W{smem, cg::this_cluster(), A.CT, 0, 0, 0, 0, 0};
    W.bulk = A.bulk;
    W.pbars = pbars;
    W.me = (int)W.cl.block_rank();
    W.lane = threadIdx.x & 31; W.sub = W.lane / TVL; W.sl = W.lane % TVL; W.warp = threadIdx.x >> 5;
    const int me = W.me;
    mbar_wait(&bar, 0);
    {
        T* b0 = sp<T>(smem, L[0].o_b);
        for (int32_t i = L[0].r0 + threadIdx.x; i < L[0].r1; i += TB) b0[i - L[0].r0] = A.b_top[i];
    }
    int tix = 0;
    auto sync = [&]() {
        W.cl.sync();
        if (A.trace && me == 0 && threadIdx.x == 0 && tix < 64) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            A.trace[tix] = t;
        }
        ++tix;
    };
    sync();  // every CTA of the cluster is resident and loaded before the first DSMEM store
    const int KT = A.KT, nu = A.nu;
    uint32_t cur[TAIL_MAXL];   // buffer holding the pre-smoothed x of each level after the down phase
    // ---------------------------------------------------------------- down
    {   // x_1 = omega_0 D^-1 b on the first tail level (own rows) -> every CTA's X
        const TailLevel& D = L[0];
        const T* b = sp<T>(smem, D.o_b);
        const T* d = sp<T>(smem, D.o_dinv);
        const int32_t own = D.r1 - D.r0;
        const int fan = W.bulk ? 1 : A.CT;
        for (int q = threadIdx.x; q < own * fan; q += TB) {
            const int32_t i = q / fan;
            const T y = (T)(A.sm_omega[0][0] * (double)d[i] * (double)b[i]);
            if (W.bulk) sp<T>(smem, D.o_X)[D.r0 + i] = y;
            else W.bcast_elem(D.o_X, D.r0 + i, y, q % A.CT);
        }
        if (W.bulk) W.publish(D, D.o_X);
        else sync();
    }
    for (int t = 0; t + 1 < KT; ++t) {
        const TailLevel& D = L[t];
        const T* b = sp<T>(smem, D.o_b);
        const T* d = sp<T>(smem, D.o_dinv);
        uint32_t in = D.o_X, out = D.o_Y;
        for (int s = 1; s < nu; ++s) {   // pre-smoothing steps 1..nu-1 (step 0 = x_1 above / in restrict)
            const double om = A.sm_omega[t][s], al = A.sm_alpha[t][s];
            for (int32_t base = D.r0 + W.warp * TRPW; base < D.r1; base += TWARPS * TRPW) {
                const int32_t i = base + W.sub;
                const bool valid = i < D.r1;
                const double sum = W.row_sum(D, valid, i, in);
                if (valid) {
                    const int32_t li = i - D.r0;
                    const double xi = (double)sp<T>(smem, in)[i];
                    double y = xi + om * (double)d[li] * ((double)b[li] - sum);
                    if (al != 0.0) y += al * (xi - (s == 1 ? 0.0 : (double)sp<T>(smem, out)[i]));
                    W.put(out, i, (T)y);
                }
            }
            if (W.bulk) W.publish(D, out);
            else sync();
            const uint32_t tt = in; in = out; out = tt;
        }
        cur[t] = in;
        // residual * P -> the owner of the aggregate's slot (one DSMEM store per row)
        {
            const T* P = sp<T>(smem, D.o_P);
            const int32_t* push = sp<int32_t>(smem, D.o_push);
            for (int32_t base = D.r0 + W.warp * TRPW; base < D.r1; base += TWARPS * TRPW) {
                const int32_t i = base + W.sub;
                const bool valid = i < D.r1;
                const double sum = W.row_sum(D, valid, i, in);
                if (valid && W.sl == 0) {
                    const int32_t li = i - D.r0;
                    const int32_t code = push[li];
                    T* dst = sp<T>(smem, D.o_slot) + (code & 0xFFFFFF);
                    *W.cl.map_shared_rank(dst, (unsigned)code >> 24) = (T)((double)P[li] * ((double)b[li] - sum));
                }
            }
            sync();
        }
        // restriction over the own aggregates (members ascending) = own rows of level t+1
        {
            const TailLevel& N = L[t + 1];
            const int64_t* mp = sp<int64_t>(smem, D.o_mp);
            const T* slot = sp<T>(smem, D.o_slot);
            T* bn = sp<T>(smem, N.o_b);
            const bool coarsest = t + 2 == KT;
            const T* dn = coarsest ? nullptr : sp<T>(smem, N.o_dinv);
            const double om0 = A.sm_omega[t + 1][0];
            for (int32_t base = D.a0 + W.warp * TRPW; base < D.a1; base += TWARPS * TRPW) {
                const int32_t a = base + W.sub;
                double sum = 0.0;
                if (a < D.a1) {
                    const int64_t s0 = mp[a - D.a0] - D.m0, s1 = mp[a - D.a0 + 1] - D.m0;
                    for (int64_t q = s0 + W.sl; q < s1; q += TVL) sum += (double)slot[q];
                }
                sum = group_sum<TVL>(sum);
                if (a < D.a1) {
                    if (W.sl == 0) bn[a - N.r0] = (T)sum;
                    // next level: its first smoothing step x_1 = omega_0 D^-1 b (or, coarsest, b itself)
                    const T y = coarsest ? (T)sum : (T)(om0 * (double)dn[a - N.r0] * sum);
                    W.put(N.o_X, a, y);
                }
            }
            if (W.bulk) W.publish(N, N.o_X);
            else sync();
        }
    }
    // ---------------------------------------------------------------- coarsest: z = A_c^-1 b (fp64 rows)
    {
        const TailLevel& C = L[KT - 1];
        const double* Ai = sp<double>(smem, C.o_Ainv);
        const T* bc = sp<T>(smem, C.o_X);
        for (int32_t i = C.r0 + W.warp; i < C.r1; i += TWARPS) {
            double s = 0.0;
            for (int32_t j = W.lane; j < C.n; j += 32) s += Ai[(int64_t)(i - C.r0) * C.n + j] * (double)bc[j];
            s = group_sum<32>(s);
            // 32 lanes share the CT stores
            const T zi = (T)s;
            if (W.bulk) { if (W.lane == 0) sp<T>(smem, C.o_Y)[i] = zi; }
            else for (int r = W.lane; r < A.CT; r += 32) W.bcast_elem(C.o_Y, i, zi, r);
        }
        if (W.bulk) W.publish(C, C.o_Y);
        else sync();
    }
    // ---------------------------------------------------------------- up
    uint32_t zbuf = L[KT - 1].o_Y;   // full z of the level below
    for (int t = KT - 2; t >= 0; --t) {
        const TailLevel& D = L[t];
        const T* b = sp<T>(smem, D.o_b);
        const T* d = sp<T>(smem, D.o_dinv);
        const T* P = sp<T>(smem, D.o_P);
        const int32_t* agg = sp<int32_t>(smem, D.o_agg);
        const T* zc = sp<T>(smem, zbuf);
        const uint32_t c0 = cur[t], other = c0 == D.o_X ? D.o_Y : D.o_X;
        {   // prolongation x_0 = x + P z_c[agg] (own rows) -> every CTA
            const int32_t own = D.r1 - D.r0;
            const T* xc = sp<T>(smem, c0);
            const int fan = W.bulk ? 1 : A.CT;
            for (int q = threadIdx.x; q < own * fan; q += TB) {
                const int32_t li = q / fan;
                const T y = (T)((double)xc[D.r0 + li] + (double)P[li] * (double)zc[agg[li]]);
                if (W.bulk) sp<T>(smem, other)[D.r0 + li] = y;
                else W.bcast_elem(other, D.r0 + li, y, q % A.CT);
            }
            if (W.bulk) W.publish(D, other);
            else sync();
        }
        uint32_t in = other, out = c0;
        for (int s = 0; s < nu; ++s) {
            const double om = A.sm_omega[t][s], al = A.sm_alpha[t][s];
            const bool last = s == nu - 1;
            for (int32_t base = D.r0 + W.warp * TRPW; base < D.r1; base += TWARPS * TRPW) {
                const int32_t i = base + W.sub;
                const bool valid = i < D.r1;
                const double sum = W.row_sum(D, valid, i, in);
                if (valid) {
                    const int32_t li = i - D.r0;
                    const double xi = (double)sp<T>(smem, in)[i];
                    double y = xi + om * (double)d[li] * ((double)b[li] - sum);
                    if (al != 0.0 && s > 0) y += al * (xi - (double)sp<T>(smem, out)[i]);
                    if (last && t == 0) {
                        if (W.sl == 0) A.z_top[i] = (T)y;
                    } else {
                        W.put(out, i, (T)y);
                    }
                }
            }
            if (!(last && t == 0)) {
                if (W.bulk) W.publish(D, out);
                else sync();
            }
            const uint32_t tt = in; in = out; out = tt;
        }
        zbuf = in;   // the buffer the last step wrote
    }
    // bulk mode: every outgoing copy has landed (each receiver waited for it) before any CTA's shared memory,
    // the copies' source, goes away
    if (W.bulk) W.cl.sync();
}


}  // namespace tail_detail
}  // namespace mgpbd
