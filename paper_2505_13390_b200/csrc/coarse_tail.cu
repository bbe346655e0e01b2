// Tail of the coarse V-cycle on one thread-block cluster, see coarse_tail.cuh.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "coarse_tail.cuh"
#include "comm.cuh"
#include "tma.cuh"
#include "util.cuh"

namespace cg = cooperative_groups;

namespace mgpbd {

namespace {

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

template <class T>
__global__ void __launch_bounds__(TB, 1) k_coarse_tail(const __grid_constant__ TailArgs<T> A) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ TailLevel L[TAIL_MAXL];
    Tail<T> W{smem, cg::this_cluster(), A.CT, 0, 0, 0, 0, 0};
    W.me = (int)W.cl.block_rank();
    W.lane = threadIdx.x & 31; W.sub = W.lane / TVL; W.sl = W.lane % TVL; W.warp = threadIdx.x >> 5;
    const int me = W.me;
    {
        const int* src = reinterpret_cast<const int*>(A.lv + (size_t)me * TAIL_MAXL);
        int* dst = reinterpret_cast<int*>(L);
        for (int k = threadIdx.x; k < (int)(TAIL_MAXL * sizeof(TailLevel) / sizeof(int)); k += TB) dst[k] = src[k];
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&bar, A.txbytes[me]);
        const TailCopy* cp = A.copies + (size_t)me * TAIL_MAXC;
        for (int k = 0; k < A.ncopies[me]; ++k) bulk_g2s(smem + cp[k].dst, cp[k].src, cp[k].bytes, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
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
        for (int q = threadIdx.x; q < own * A.CT; q += TB) {
            const int32_t i = q / A.CT;
            const T y = (T)(A.sm_omega[0][0] * (double)d[i] * (double)b[i]);
            W.bcast_elem(D.o_X, D.r0 + i, y, q % A.CT);
        }
        sync();
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
                    W.bcast_row(out, i, (T)y);
                }
            }
            sync();
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
                    W.bcast_row(N.o_X, a, y);
                }
            }
            sync();
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
            for (int r = W.lane; r < A.CT; r += 32) W.bcast_elem(C.o_Y, i, zi, r);
        }
        sync();
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
            for (int q = threadIdx.x; q < own * A.CT; q += TB) {
                const int32_t li = q / A.CT;
                const T y = (T)((double)xc[D.r0 + li] + (double)P[li] * (double)zc[agg[li]]);
                W.bcast_elem(other, D.r0 + li, y, q % A.CT);
            }
            sync();
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
                        W.bcast_row(out, i, (T)y);
                    }
                }
            }
            if (!(last && t == 0)) sync();
            const uint32_t tt = in; in = out; out = tt;
        }
        zbuf = in;   // the buffer the last step wrote
    }
}

}  // namespace

template <class T>
bool coarse_tail_launchable(int CT, uint32_t smem) {
    if (!try_raise_dyn_smem((const void*)k_coarse_tail<T>, smem)) return false;
    if (CT > 8 && cudaFuncSetAttribute((const void*)k_coarse_tail<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                      cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CT);
    cfg.blockDim = dim3(TB);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CT; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (const void*)k_coarse_tail<T>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return nc >= 1;
}

template <class T>
bool coarse_tail_plan(const CoarseCycle<T>& c, int min_first, int CT, uint32_t smem_cap, TailPlan& plan, cudaStream_t s) {
    const int K = c.K;
    if (K < 2 || K - min_first < 2) return false;
    // host copies of the static structure of every candidate level
    std::vector<std::vector<int64_t>> rp(K), mp(K);
    std::vector<std::vector<int32_t>> col(K), agg(K), ml(K);
    for (int k = std::max(min_first, 0); k < K; ++k) {
        const CoarseLevel<T>& L = c.L[k];
        if (k + 1 < K) {
            rp[k].resize((size_t)L.n + 1);
            d2h(rp[k].data(), L.rowptr, (size_t)L.n + 1, s);
            MG_CK(cudaStreamSynchronize(s));
            col[k].resize((size_t)rp[k][L.n]);
            d2h(col[k].data(), L.col, col[k].size(), s);
            agg[k].resize(L.n);
            d2h(agg[k].data(), L.agg, (size_t)L.n, s);
            mp[k].resize((size_t)L.n_agg + 1);
            d2h(mp[k].data(), L.mptr, (size_t)L.n_agg + 1, s);
            MG_CK(cudaStreamSynchronize(s));
            ml[k].resize((size_t)mp[k][L.n_agg]);
            d2h(ml[k].data(), L.mlist, ml[k].size(), s);
        }
    }
    MG_CK(cudaStreamSynchronize(s));
    const size_t ts = sizeof(T);
    for (int first = std::max(min_first, 1); first + 1 < K; ++first) {
        const int KT = K - first;
        if (KT > TAIL_MAXL) continue;
        bool fits16 = true;
        for (int k = first; k + 1 < K; ++k) fits16 = fits16 && c.L[k].n <= 65536;
        if (!fits16) continue;
        // row partitions: nnz-balanced (coarsest: even)
        std::vector<std::vector<int32_t>> rb(KT);
        for (int t = 0; t < KT; ++t) {
            const int k = first + t;
            if (k + 1 < K) rb[t] = partition_rows(rp[k].data(), c.L[k].n, CT);
            else {
                rb[t].resize(CT + 1);
                for (int g = 0; g <= CT; ++g) rb[t][g] = (int32_t)((int64_t)c.L[k].n * g / CT);
            }
        }
        // smem layout per CTA
        std::vector<TailLevel> lv((size_t)CT * TAIL_MAXL);
        std::vector<TailCopy> cps((size_t)CT * TAIL_MAXC, TailCopy{nullptr, 0, 0});
        std::vector<int32_t> ncp(CT, 0);
        std::vector<uint32_t> tx(CT, 0);
        uint32_t smem = 0;
        bool ok = true;
        // device images: 16-bit columns and push codes (built once per plan attempt that fits)
        std::vector<std::vector<uint16_t>> c16(KT);
        std::vector<std::vector<int32_t>> push(KT);
        for (int t = 0; t + 1 < KT; ++t) {
            const int k = first + t;
            c16[t].resize(col[k].size());
            for (size_t e = 0; e < col[k].size(); ++e) c16[t][e] = (uint16_t)col[k][e];
            // slot of each row in the member list; owner of its aggregate = row owner on level t+1
            std::vector<int64_t> slot(c.L[k].n);
            for (int64_t q = 0; q < (int64_t)ml[k].size(); ++q) slot[ml[k][q]] = q;
            push[t].resize(c.L[k].n);
            for (int32_t i = 0; i < c.L[k].n; ++i) {
                const int32_t a = agg[k][i];
                const int g = (int)(std::upper_bound(rb[t + 1].begin(), rb[t + 1].end(), a) - rb[t + 1].begin()) - 1;
                const int64_t off = slot[i] - mp[k][rb[t + 1][g]];
                push[t][i] = (int32_t)(((uint32_t)g << 24) | (uint32_t)off);
                if (off >= (1 << 24)) ok = false;
            }
        }
        if (!ok) continue;
        for (int t = 0; t + 1 < KT; ++t) {
            plan.col16[t].resize(c16[t].size());
            h2d(plan.col16[t].p, c16[t].data(), c16[t].size(), s);
            plan.push[t].resize(push[t].size());
            h2d(plan.push[t].p, push[t].data(), push[t].size(), s);
        }
        // buffers other CTAs store into (DSMEM addresses are the same smem offset in every CTA): the full
        // X / Y vectors of every level and the restriction slot arrays, at common offsets first
        uint32_t common = 0;
        std::vector<uint32_t> oX(KT), oY(KT), oS(KT, 0);
        auto common_alloc = [&](uint32_t& off, size_t bytes) {
            off = (common + 15u) & ~15u;
            common = off + (uint32_t)bytes;
        };
        for (int t = 0; t < KT; ++t) {
            const int k = first + t;
            common_alloc(oX[t], (size_t)c.L[k].n * ts);
            common_alloc(oY[t], (size_t)c.L[k].n * ts);
            if (t + 1 < KT) {
                int64_t mx = 0;
                for (int g = 0; g < CT; ++g) mx = std::max(mx, mp[k][rb[t + 1][g + 1]] - mp[k][rb[t + 1][g]]);
                common_alloc(oS[t], (size_t)mx * ts);
            }
        }
        for (int g = 0; g < CT && ok; ++g) {
            uint32_t cursor = common;
            int nc = 0;
            auto add = [&](uint32_t& off, const void* base, int64_t elem_off, size_t esz, size_t count) -> bool {
                const uintptr_t src = reinterpret_cast<uintptr_t>(base) + (uintptr_t)(elem_off * (int64_t)esz);
                const uintptr_t al = src & ~(uintptr_t)15;
                const uint32_t lead = (uint32_t)(src - al);
                const uint32_t dst = (cursor + 15u) & ~15u;
                off = dst + lead;   // the kernel indexes own-range arrays locally (element elem_off at off)
                const size_t bytes = count * esz;
                if (bytes == 0) { cursor = dst + lead; return true; }
                const uint32_t nb = (uint32_t)((lead + bytes + 15) & ~(size_t)15);
                if (nc >= TAIL_MAXC) return false;
                cps[(size_t)g * TAIL_MAXC + nc++] = TailCopy{reinterpret_cast<const void*>(al), dst, nb};
                cursor = dst + nb;
                tx[g] += nb;
                return true;
            };
            auto alloc = [&](uint32_t& off, size_t esz, size_t count) {
                const uint32_t dst = (cursor + 15u) & ~15u;
                off = dst;
                cursor = dst + (uint32_t)(count * esz);
            };
            for (int t = 0; t < KT && ok; ++t) {
                const int k = first + t;
                const CoarseLevel<T>& Lk = c.L[k];
                TailLevel& d = lv[(size_t)g * TAIL_MAXL + t];
                d.n = Lk.n;
                d.r0 = rb[t][g]; d.r1 = rb[t][g + 1];
                const int64_t rows = d.r1 - d.r0;
                if (t + 1 < KT) {
                    d.e0 = rp[k][d.r0];
                    const int64_t nnz = rp[k][d.r1] - d.e0;
                    d.a0 = rb[t + 1][g]; d.a1 = rb[t + 1][g + 1];
                    d.m0 = mp[k][d.a0];
                    const int64_t mem = mp[k][d.a1] - d.m0;
                    // element-0-relative offsets: o_x + elem * size addresses element elem
                    ok = ok && add(d.o_rp, Lk.rowptr, d.r0, 8, (size_t)rows + 1);
                    ok = ok && add(d.o_col, plan.col16[t].p, d.e0, 2, (size_t)nnz);
                    ok = ok && add(d.o_val, Lk.val, d.e0, ts, (size_t)nnz);
                    ok = ok && add(d.o_dinv, Lk.dinv, d.r0, ts, (size_t)rows);
                    ok = ok && add(d.o_P, Lk.P, d.r0, ts, (size_t)rows);
                    ok = ok && add(d.o_agg, Lk.agg, d.r0, 4, (size_t)rows);
                    ok = ok && add(d.o_push, plan.push[t].p, d.r0, 4, (size_t)rows);
                    ok = ok && add(d.o_mp, Lk.mptr, d.a0, 8, (size_t)(d.a1 - d.a0) + 1);
                    (void)mem;
                    d.o_slot = oS[t];
                    if (t == 0) ok = ok && add(d.o_b, Lk.b, d.r0, ts, (size_t)rows);
                    else alloc(d.o_b, ts, (size_t)rows);
                } else {
                    ok = ok && add(d.o_Ainv, c.Ainv, (int64_t)d.r0 * Lk.n, 8, (size_t)rows * Lk.n);
                    alloc(d.o_b, ts, (size_t)rows);
                }
                d.o_X = oX[t];   // full-length vectors (global row index), common offsets
                d.o_Y = oY[t];
            }
            ncp[g] = nc;
            smem = std::max(smem, cursor);
            if (cursor > smem_cap) ok = false;
        }
        if (!ok) continue;
        plan.first = first;
        plan.CT = CT;
        plan.smem = smem;
        plan.lv.resize(lv.size()); h2d(plan.lv.p, lv.data(), lv.size(), s);
        plan.copies.resize(cps.size()); h2d(plan.copies.p, cps.data(), cps.size(), s);
        plan.ncopies.resize(ncp.size()); h2d(plan.ncopies.p, ncp.data(), ncp.size(), s);
        plan.txbytes.resize(tx.size()); h2d(plan.txbytes.p, tx.data(), tx.size(), s);
        MG_CK(cudaStreamSynchronize(s));
        return true;
    }
    return false;
}

template <class T>
void coarse_tail_run(const CoarseCycle<T>& c, const TailPlan& plan, cudaStream_t s) {
    TailArgs<T> a;
    a.KT = c.K - plan.first;
    a.nu = c.nu;
    a.CT = plan.CT;
    a.lv = plan.lv.p;
    a.copies = plan.copies.p;
    a.ncopies = plan.ncopies.p;
    a.txbytes = plan.txbytes.p;
    a.b_top = c.L[plan.first].b;
    a.z_top = c.L[plan.first].z;
    for (int t = 0; t < a.KT && t < TAIL_MAXL; ++t)
        for (int q = 0; q < 8; ++q) {
            a.sm_omega[t][q] = c.L[plan.first + t].sm_omega[q];
            a.sm_alpha[t][q] = c.L[plan.first + t].sm_alpha[q];
        }
    a.trace = c.trace ? c.trace + 32 : nullptr;
    ensure_dyn_smem((const void*)k_coarse_tail<T>, plan.smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.CT);
    cfg.blockDim = dim3(TB);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = plan.CT; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MG_CK(cudaLaunchKernelEx(&cfg, k_coarse_tail<T>, a));
    MG_LAUNCH_CHECK();
}

#define MG_INST(T)                                                                                               \
    template bool coarse_tail_plan<T>(const CoarseCycle<T>&, int, int, uint32_t, TailPlan&, cudaStream_t);     \
    template bool coarse_tail_launchable<T>(int, uint32_t);                                                      \
    template void coarse_tail_run<T>(const CoarseCycle<T>&, const TailPlan&, cudaStream_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
