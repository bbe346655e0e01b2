// Tail of the coarse V-cycle on one thread-block cluster, see coarse_tail.cuh.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "coarse_tail.cuh"
#include "coarse_tail_body.cuh"
#include "comm.cuh"
#include "tma.cuh"
#include "util.cuh"

namespace cg = cooperative_groups;

namespace mgpbd {

namespace {

constexpr int TB = tail_detail::TB;

template <class T>
__global__ void __launch_bounds__(TB, 1) k_coarse_tail(const __grid_constant__ TailArgs<T> A) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ TailLevel L[TAIL_MAXL];
    __shared__ __align__(8) uint64_t pbars[2];
    tail_detail::coarse_tail_load<T>(A, smem, L, bar, pbars);
    tail_detail::coarse_tail_body<T>(A, smem, L, bar, pbars);
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
        // row partitions: nnz-balanced (coarsest: even), interior bounds rounded to 16-byte multiples so every
        // CTA's own range can be broadcast as one bulk copy
        const int32_t VEC = (int32_t)(16 / ts);
        std::vector<std::vector<int32_t>> rb(KT);
        for (int t = 0; t < KT; ++t) {
            const int k = first + t;
            if (k + 1 < K) rb[t] = partition_rows(rp[k].data(), c.L[k].n, CT);
            else {
                rb[t].resize(CT + 1);
                for (int g = 0; g <= CT; ++g) rb[t][g] = (int32_t)((int64_t)c.L[k].n * g / CT);
            }
            for (int g = 1; g < CT; ++g)
                rb[t][g] = std::max(rb[t][g - 1], std::min(c.L[k].n, (rb[t][g] + VEC / 2) / VEC * VEC));
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
            const size_t npad = ((size_t)c.L[k].n + VEC - 1) / VEC * VEC;   // the last CTA's range rounds up
            common_alloc(oX[t], npad * ts);
            common_alloc(oY[t], npad * ts);
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
                    alloc(d.o_b, ts, (size_t)rows);   // t = 0: read from b_top by the kernel (not static)
                } else {
                    ok = ok && add(d.o_Ainv, c.Ainv, (int64_t)d.r0 * Lk.n, 8, (size_t)rows * Lk.n);
                    alloc(d.o_b, ts, (size_t)rows);
                }
                d.o_X = oX[t];   // full-length vectors (global row index), common offsets
                d.o_Y = oY[t];
                auto obytes = [&](int gg) {
                    const int32_t a = rb[t][gg], b = rb[t][gg + 1];
                    return (uint32_t)(((int64_t)(b - a) * (int64_t)ts + 15) & ~(int64_t)15);
                };
                d.ob = obytes(g);
                d.rx = 0;
                for (int gg = 0; gg < CT; ++gg)
                    if (gg != g) d.rx += obytes(gg);
            }
            ncp[g] = nc;
            smem = std::max(smem, cursor);
            if (cursor > smem_cap) ok = false;
        }
        if (!ok) continue;
        plan.first = first;
        plan.CT = CT;
        plan.bulk = std::getenv("MGPBD_TAIL_SCALAR_BCAST") ? 0 : 1;
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
TailArgs<T> coarse_tail_args(const CoarseCycle<T>& c, const TailPlan& plan) {
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
    a.bulk = plan.bulk;
    return a;
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
    a.bulk = plan.bulk;
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
    template void coarse_tail_run<T>(const CoarseCycle<T>&, const TailPlan&, cudaStream_t);                     \
    template TailArgs<T> coarse_tail_args<T>(const CoarseCycle<T>&, const TailPlan&);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
