// Matrix-free level-0 operator, see matfree.cuh.
#include <algorithm>
#include <cstring>
#include <type_traits>
#include <vector>

#include "matfree.cuh"
#include "tma.cuh"
#include "util.cuh"
#include "record.cuh"
#include "solve.cuh"

namespace mgpbd {

namespace {

constexpr int MF_BS = 256;
#ifndef MGPBD_MF_R
#define MGPBD_MF_R 128  // swept on B200 (profiles/r1/sweep_level0_pass.txt): 128 rows, 3 stages, 6 CTAs/SM
#endif
constexpr int MF_R = MGPBD_MF_R;  // rows per tile (= threads per CTA) of tetrahedra
#ifndef MGPBD_MF_R2
#define MGPBD_MF_R2 256  // fp32 distance constraints (2 vertices per row), swept on cloth2048 (profiles/r2):
#endif                   // 220 us per pass vs 228 (128 rows) and 237 (512); fp64 keeps 128 (429 vs 463 us)
template <class T, int KC>
__host__ __device__ constexpr int mf_r() { return (KC == 2 && sizeof(T) == 4) ? MGPBD_MF_R2 : MF_R; }
inline int mf_r(int kc, int tsize) { return (kc == 2 && tsize == 4) ? MGPBD_MF_R2 : MF_R; }
#ifndef MGPBD_MF_STAGES
#define MGPBD_MF_STAGES 3
#endif
constexpr int MF_STAGES = MGPBD_MF_STAGES;  // ring depth (overridable at build time for tuning sweeps)

template <class T>
struct alignas(4 * sizeof(T)) V4 {
    T x, y, z, w;
};

// hv[plane][p] = h[vsrc[p]][plane] (0 on pad slots) for the padded slots [p0, p1) of the vertices
// [v0, v1); at_i = alpha_i / dt^2 for all rows; dinv_i = 1 / (sum_s |h_{i,s}|^2 + at_i) for rows [r0, r1) —
// the assembly's diagonal formula (mesh.cu k_assemble), so the smoother does not need the assembled matrix.
template <class T, int KC>
__global__ void k_mf_refresh(int64_t p0, int64_t p1, int64_t npad, const int32_t* __restrict__ vsrc,
                             const T* __restrict__ h, T* __restrict__ hv, int32_t m, int32_t r0, int32_t r1,
                             const double* __restrict__ alpha, double dt2, T* __restrict__ at,
                             T* __restrict__ dinv) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = p0 + tid; p < p1; p += nt) {
        const int32_t code = vsrc[p];
        const T* q = h + (int64_t)(code < 0 ? 0 : code) * 3;
        hv[p] = code < 0 ? (T)0 : q[0];
        hv[npad + p] = code < 0 ? (T)0 : q[1];
        hv[2 * npad + p] = code < 0 ? (T)0 : q[2];
    }
    for (int64_t i = tid; i < m; i += nt) {
        const double a = alpha[i] / dt2;
        at[i] = (T)a;
        if (i >= r0 && i < r1) {
            T hi[KC][3];
            load_record<T, KC>(h + i * KC * 3, hi);
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < KC; ++k)
                d += (double)hi[k][0] * hi[k][0] + (double)hi[k][1] * hi[k][1] + (double)hi[k][2] * hi[k][2];
            d += a;
            dinv[i] = (T)(1.0 / (double)(T)d);
        }
    }
}

// timing experiments only (tools/pass_sweep.sh; results are wrong): 1 = no x gather in the vertex gather,
// 2 = no h planes (only the constraint offsets streamed)
#ifndef MGPBD_VG_EXPT
#define MGPBD_VG_EXPT 0
#endif
// One 16-byte chunk of a vertex's padded incidence list: VW = 16 / sizeof(T) incidences of the three h planes
// and their constraint indices (16- or 32-bit).
template <class T, bool J16>
struct Chunk {
    static constexpr int VW = 16 / (int)sizeof(T);
    T hx[VW], hy[VW], hz[VW];
    int32_t j[VW];
    // SM: the chunk lives in shared memory (plain loads); otherwise global, streamed (evict-first)
    // POL: global loads carry the L2 policy `pol` (MGPBD_L2POL) instead of the streaming hint
    template <bool SM = false, bool POL = false>
    __device__ __forceinline__ void load(const T* __restrict__ hx_, const T* __restrict__ hy_, const T* __restrict__ hz_,
                                         const uint16_t* __restrict__ j16, const int32_t* __restrict__ j32, int64_t p,
                                         bool in, uint64_t pol = 0) {
        using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
        auto ld = [pol](const auto* q) {
            using Q = typename std::remove_cv<typename std::remove_pointer<decltype(q)>::type>::type;
            if constexpr (SM) {
                return *q;
            } else if constexpr (POL) {
                Q r;
                if constexpr (sizeof(Q) == 16) { const uint4 w = ldg16_pol(q, pol); memcpy(&r, &w, 16); }
                else if constexpr (sizeof(Q) == 8) { const uint2 w = ldg8_pol(q, pol); memcpy(&r, &w, 8); }
                else { const uint32_t w = ldg4_pol(q, pol); memcpy(&r, &w, 4); }
                return r;
            } else {
                return __ldcs(q);
            }
        };
        if (in) {
            if (MGPBD_VG_EXPT == 2 && !SM) {
#pragma unroll
                for (int w = 0; w < VW; ++w) hx[w] = hy[w] = hz[w] = (T)(p + w);
            } else {
                const VT a = ld(reinterpret_cast<const VT*>(hx_ + p));
                const VT b = ld(reinterpret_cast<const VT*>(hy_ + p));
                const VT c = ld(reinterpret_cast<const VT*>(hz_ + p));
                memcpy(hx, &a, 16); memcpy(hy, &b, 16); memcpy(hz, &c, 16);
            }
            if constexpr (J16 && VW == 4) {
                const uint2 w = ld(reinterpret_cast<const uint2*>(j16 + p));
                j[0] = (int32_t)(w.x & 0xFFFFu); j[1] = (int32_t)(w.x >> 16);
                j[2] = (int32_t)(w.y & 0xFFFFu); j[3] = (int32_t)(w.y >> 16);
            } else if constexpr (J16) {
                const unsigned int w = ld(reinterpret_cast<const unsigned int*>(j16 + p));
                j[0] = (int32_t)(w & 0xFFFFu); j[1] = (int32_t)(w >> 16);
            } else if constexpr (VW == 4) {
                const int4 w = ld(reinterpret_cast<const int4*>(j32 + p));
                j[0] = w.x; j[1] = w.y; j[2] = w.z; j[3] = w.w;
            } else {
                const int2 w = ld(reinterpret_cast<const int2*>(j32 + p));
                j[0] = w.x; j[1] = w.y;
            }
        } else {
#pragma unroll
            for (int w = 0; w < VW; ++w) { hx[w] = hy[w] = hz[w] = (T)0; j[w] = 0; }
        }
    }
};

// u_v = sum over v's incidences of h_{j,s} x_j over the padded vertex-major layout: G lanes per vertex, each
// lane streams 16-byte chunks (UN per round: all loads, then all x gathers, then the sums), fixed butterfly
// (deterministic).  Accumulation in the storage precision unless MGPBD_VG_ACC64 (fp32 -> fp64 conversions
// are quarter-rate on sm_100a; DESIGN.md §2 reading c18 records the measured cost and parity impact).
#ifndef MGPBD_VG_ACC64
#define MGPBD_VG_ACC64 0
#endif
// XJ: x is not materialised — x_j = omega0 D^-1_jj b_j (the V-cycle's first smoothing step from x = 0,
// k_jacobi0's expression), gathered from dinv and b.
#ifndef MGPBD_VG_MINB
#define MGPBD_VG_MINB 1
#endif
#ifndef MGPBD_VG_PREFETCH
#define MGPBD_VG_PREFETCH 1
#endif
// 2 (default): contiguous vertex range per CTA of a persistent grid (x values reused from L1 across the
// constraints a vertex plane shares with the next: 45.9 -> 43.4 us per fp32 pass, profiles/r2/experiments_log.txt);
// 1: the same with the ranges of the CTAs co-resident on an SM adjacent; 0: grid-stride
#ifndef MGPBD_VG_BLOCKED
#define MGPBD_VG_BLOCKED 2
#endif
// threads per CTA of the register vertex gather: fp32 one 1024-thread CTA per SM (its 32 warps share one contiguous
// vertex range: 41.5 -> 40.6 us per pass), fp64 256 (its 3-chunk rounds need more than 64 registers)
#ifndef MGPBD_VG_THREADS
#define MGPBD_VG_THREADS 1024
#endif
template <class T>
constexpr int vg_threads() { return sizeof(T) == 4 ? MGPBD_VG_THREADS : 256; }
// Vertices of the calling warp over [v0, v1): base = first, first + step, ... < vend (MGPBD_VG_BLOCKED: one
// contiguous range per CTA of a persistent grid, see k_mf_vgather; else grid-stride)
struct VRange {
    int64_t first, step, vend;
};
template <int PER_WARP>
__device__ __forceinline__ VRange warp_vertices(int32_t v0, int32_t v1, int nsm) {
    VRange r;
    if (MGPBD_VG_BLOCKED) {
        const int S = gridDim.x < (unsigned)nsm ? (int)gridDim.x : nsm;
        const int per = (int)gridDim.x / S;
        const int c = MGPBD_VG_BLOCKED == 2 ? (int)blockIdx.x : (int)(blockIdx.x % S) * per + (int)(blockIdx.x / S);
        const int64_t wpc = blockDim.x >> 5;
        const int64_t chunk = ((v1 - v0 + (int64_t)gridDim.x - 1) / gridDim.x + wpc * PER_WARP - 1) / (wpc * PER_WARP) * (wpc * PER_WARP);
        const int64_t cs = v0 + (int64_t)c * chunk;
        r.vend = cs + chunk < v1 ? cs + chunk : v1;
        r.first = cs + (int64_t)(threadIdx.x >> 5) * PER_WARP;
        r.step = wpc * PER_WARP;
    } else {
        const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        r.first = v0 + warp * PER_WARP;
        r.step = (((int64_t)gridDim.x * blockDim.x) >> 5) * PER_WARP;
        r.vend = v1;
    }
    return r;
}
inline int vg_sms() {
    static const int n = [] {
        int dev = 0, sms = 148;
        MG_CK(cudaGetDevice(&dev));
        MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        return sms;
    }();
    return n;
}
// L2 policy of the level-0 pass's two gradient streams (hv in the vertex gather, h in the row kernel; each
// ~80 MB fp32 on block1.67M, read 50 times per outer iteration): 0 = streaming (evict-first loads in the
// gather, default bulk copies), 1 = gather stream evict_last + row stream evict_first, 2 = the reverse,
// 3 = gather stream evict_last, row stream default.
#ifndef MGPBD_L2POL
#define MGPBD_L2POL 0
#endif
template <class T, int G, int UN, bool J16, bool XJ>
__global__ void __launch_bounds__(vg_threads<T>(), MGPBD_VG_MINB) k_mf_vgather(int32_t v0, int32_t v1, int64_t npad,
                                                      const int64_t* __restrict__ ppos,
                                                      const uint16_t* __restrict__ vj16,
                                                      const int32_t* __restrict__ vj32,
                                                      const int32_t* __restrict__ jbase, const T* __restrict__ hv,
                                                      const T* __restrict__ x, V4<T>* __restrict__ u,
                                                      const T* __restrict__ xd, const T* __restrict__ xb, double xom, int nsm) {
    using CH = Chunk<T, J16>;
    constexpr int VW = CH::VW;
    constexpr int PER_WARP = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
    // vertices of this warp: base = first, first + step, ... < vend.  Grid-stride over the whole range, or
    // (MGPBD_VG_BLOCKED, persistent grid) one contiguous range per CTA, the CTAs resident on one SM holding
    // adjacent ranges (CTA i runs on SM i mod S), so an SM sweeps ~n_v / S consecutive vertices and the x values
    // of the constraints between two vertex planes are reused from its L1
    const VRange vr = warp_vertices<PER_WARP>(v0, v1, nsm);
    const int64_t first = vr.first, step = vr.step, vend = vr.vend;
    const T* __restrict__ hx = hv;
    const T* __restrict__ hy = hv + npad;
    const T* __restrict__ hz = hv + 2 * npad;
    const uint64_t pol = MGPBD_L2POL == 1 || MGPBD_L2POL == 3 ? l2_policy_last() : MGPBD_L2POL == 2 ? l2_policy_first() : 0;
    // the next vertex's slot range and index base are fetched one round ahead (one dependent round trip less
    // per vertex)
    int64_t p0n = 0, p1n = 0;
    int32_t jbn = 0;
    auto fetch = [&](int64_t vv) {
        if (vv < vend) { p0n = ppos[vv]; p1n = ppos[vv + 1]; jbn = J16 ? jbase[vv] : 0; }
    };
    if (MGPBD_VG_PREFETCH) fetch(first + sub);
    // launched with programmatic dependent launch (MatFree::vg_pdl): everything above reads static data; x is
    // the previous kernel's output (no-op otherwise)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // programmatic dependent launch: the row kernel may start streaming its operands now (it waits in
    // griddepcontrol.wait for this grid's u before gathering it).  Released after this grid's own wait, so
    // that everything launched before it (the kernel that wrote x, b) is complete when the row kernel's
    // pre-wait prologue reads it, whichever kernel released this grid early (MG_VEC_TRIGGER, solve.cu)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int64_t base = first; base < vend; base += step) {  // warp-uniform
        const int64_t v = base + sub;
        using AC = typename std::conditional<MGPBD_VG_ACC64 != 0, double, T>::type;
        AC a0 = (AC)0, a1 = (AC)0, a2 = (AC)0;
        if (!MGPBD_VG_PREFETCH) fetch(v);
        const int64_t p0 = p0n, p1 = p1n;
        const int32_t jb = jbn;
        if (MGPBD_VG_PREFETCH) fetch(v + step);
        if (v < vend) {
            for (int64_t pb = p0 + (int64_t)sl * VW; pb < p1; pb += (int64_t)G * VW * UN) {
                CH c[UN];
#pragma unroll
                for (int q = 0; q < UN; ++q) {
                    const int64_t p = pb + (int64_t)q * G * VW;
                    c[q].template load<false, (MGPBD_L2POL != 0)>(hx, hy, hz, vj16, vj32, p, p < p1, pol);
                }
                T xv[UN][VW];
#pragma unroll
                for (int q = 0; q < UN; ++q)
#pragma unroll
                    for (int w = 0; w < VW; ++w) {
                        const int32_t jj = jb + c[q].j[w];
                        if (MGPBD_VG_EXPT == 1) xv[q][w] = (T)jj;   // timing experiment: no x gather
                        else if (XJ) xv[q][w] = (T)(xom * (double)xd[jj] * (double)xb[jj]);
                        else xv[q][w] = x[jj];
                    }
#pragma unroll
                for (int q = 0; q < UN; ++q)
#pragma unroll
                    for (int w = 0; w < VW; ++w) {
                        a0 += (AC)c[q].hx[w] * (AC)xv[q][w];
                        a1 += (AC)c[q].hy[w] * (AC)xv[q][w];
                        a2 += (AC)c[q].hz[w] * (AC)xv[q][w];
                    }
            }
        }
        a0 = group_sum_t<G>(a0);
        a1 = group_sum_t<G>(a1);
        a2 = group_sum_t<G>(a2);
        if (v < vend && sl == 0) u[v] = V4<T>{(T)a0, (T)a1, (T)a2, (T)0};
    }
}

// TMA-pipelined vertex gather: persistent CTAs stream tiles of VGT consecutive vertices — their padded slot
// ranges of the three h planes, the constraint offsets and the vertex's slot offsets — into a VG_STAGES-deep
// shared-memory ring with 1-D bulk copies, so the HBM stream never waits on the dependent x gathers; G lanes
// per vertex read 16-byte chunks from shared memory and gather x from L2 (same sums, same order as
// k_mf_vgather).
#ifndef MGPBD_VGT
#define MGPBD_VGT 32
#endif
constexpr int VGT = MGPBD_VGT;       // vertices per tile
#ifndef MGPBD_VG_BS
#define MGPBD_VG_BS 128
#endif
#ifndef MGPBD_VG_STAGES
#define MGPBD_VG_STAGES 3
#endif
constexpr int VG_BS = MGPBD_VG_BS;   // threads per CTA
constexpr int VG_STAGES = MGPBD_VG_STAGES;

template <class T, bool J16>
struct VgLayout {                    // one stage for tiles of at most TS slots
    uint32_t hx, hy, hz, j, pp, bytes;
    __host__ __device__ VgLayout(int32_t TS) {
        const uint32_t ph = (uint32_t)TS * sizeof(T);
        hx = 0; hy = ph; hz = 2 * ph; j = 3 * ph;
        const uint32_t jb = (uint32_t)TS * (J16 ? 2u : 4u) + 16u;
        pp = j + ((jb + 15u) & ~15u);
        bytes = pp + (uint32_t)((VGT + 4) * 8);
    }
};

template <class T, int G, bool J16>
__global__ void __launch_bounds__(VG_BS) k_mf_vgather_tma(int32_t v0, int32_t v1, int32_t ntiles, int32_t TS,
                                                          int64_t npad, const int64_t* __restrict__ ppos,
                                                          const uint16_t* __restrict__ vj16,
                                                          const int32_t* __restrict__ vj32,
                                                          const int32_t* __restrict__ jbase, const T* __restrict__ hv,
                                                          const T* __restrict__ x, V4<T>* __restrict__ u) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[VG_STAGES];
    const VgLayout<T, J16> LY(TS);
    const int t = threadIdx.x;
    if (t == 0) {
        for (int k = 0; k < VG_STAGES; ++k) mbar_init(&bars[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const T* __restrict__ hx = hv;
    const T* __restrict__ hy = hv + npad;
    const T* __restrict__ hz = hv + 2 * npad;
    const unsigned char* jsrc = J16 ? reinterpret_cast<const unsigned char*>(vj16) : reinterpret_cast<const unsigned char*>(vj32);
    constexpr uint32_t JB = J16 ? 2u : 4u;
    auto issue = [&](int jt) {
        const int tile = blockIdx.x + jt * gridDim.x;
        unsigned char* st = smem + (size_t)(jt % VG_STAGES) * LY.bytes;
        const int32_t va = v0 + tile * VGT, vb = min(va + VGT, v1);
        const int64_t pa = ppos[va], pb = ppos[vb];
        const uint32_t ns = (uint32_t)(pb - pa);
        const uintptr_t ja = reinterpret_cast<uintptr_t>(jsrc + pa * JB), ja0 = ja & ~(uintptr_t)15;
        const uint32_t jbytes = (uint32_t)(((ja - ja0) + (uintptr_t)ns * JB + 15) & ~(uintptr_t)15);
        const uintptr_t pp = reinterpret_cast<uintptr_t>(ppos + va), pp0 = pp & ~(uintptr_t)15;
        const uint32_t pbytes = (uint32_t)(((pp - pp0) + (uintptr_t)(vb - va + 1) * 8 + 15) & ~(uintptr_t)15);
        uint64_t* bar = &bars[jt % VG_STAGES];
        mbar_expect_tx(bar, 3 * ns * (uint32_t)sizeof(T) + jbytes + pbytes);
        if (ns) {
            bulk_g2s(st + LY.hx, hx + pa, ns * (uint32_t)sizeof(T), bar);
            bulk_g2s(st + LY.hy, hy + pa, ns * (uint32_t)sizeof(T), bar);
            bulk_g2s(st + LY.hz, hz + pa, ns * (uint32_t)sizeof(T), bar);
        }
        bulk_g2s(st + LY.j, reinterpret_cast<const void*>(ja0), jbytes, bar);
        bulk_g2s(st + LY.pp, reinterpret_cast<const void*>(pp0), pbytes, bar);
    };
    const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (t == 0)
        for (int jt = 0; jt < VG_STAGES && jt < my_tiles; ++jt) issue(jt);
    using CH = Chunk<T, J16>;
    constexpr int VW = CH::VW;
    const int g = t / G, sl = t % G;
    for (int jt = 0; jt < my_tiles; ++jt) {
        mbar_wait(&bars[jt % VG_STAGES], (uint32_t)((jt / VG_STAGES) & 1));
        const unsigned char* st = smem + (size_t)(jt % VG_STAGES) * LY.bytes;
        const int tile = blockIdx.x + jt * gridDim.x;
        const int32_t va = v0 + tile * VGT, vb = min(va + VGT, v1);
        const uintptr_t pp = reinterpret_cast<uintptr_t>(ppos + va);
        const int64_t* spp = reinterpret_cast<const int64_t*>(st + LY.pp) + ((pp & 15) >> 3);
        const int64_t pa = spp[0];
        const uint32_t jlead = (uint32_t)(reinterpret_cast<uintptr_t>(jsrc + pa * JB) & 15);
        const T* shx = reinterpret_cast<const T*>(st + LY.hx);
        const T* shy = reinterpret_cast<const T*>(st + LY.hy);
        const T* shz = reinterpret_cast<const T*>(st + LY.hz);
        const unsigned char* sj = st + LY.j + jlead;
        for (int vi = g; vi < VGT; vi += VG_BS / G) {   // uniform trip count: the butterfly needs the group
            const int32_t v = va + vi;
            T a0 = (T)0, a1 = (T)0, a2 = (T)0;
            if (v < vb) {
                const int64_t s0 = spp[vi] - pa, s1 = spp[vi + 1] - pa;
                const int32_t jb = J16 ? jbase[v] : 0;
                // rounds of VUN chunks per lane: all chunks from shared memory, then all their x gathers (one L2
                // round trip per round), then the products
                constexpr int VUN = 2;
                for (int64_t sb = s0 + (int64_t)sl * VW; sb < s1; sb += (int64_t)G * VW * VUN) {
                    CH c[VUN];
#pragma unroll
                    for (int q = 0; q < VUN; ++q) {
                        const int64_t sq = sb + (int64_t)q * G * VW;
                        c[q].template load<true>(shx, shy, shz, reinterpret_cast<const uint16_t*>(sj),
                                                 reinterpret_cast<const int32_t*>(sj), sq, sq < s1);
                    }
                    T xv[VUN][VW];
#pragma unroll
                    for (int q = 0; q < VUN; ++q)
#pragma unroll
                        for (int w = 0; w < VW; ++w) xv[q][w] = x[jb + c[q].j[w]];
#pragma unroll
                    for (int q = 0; q < VUN; ++q)
#pragma unroll
                        for (int w = 0; w < VW; ++w) {
                            a0 += c[q].hx[w] * xv[q][w];
                            a1 += c[q].hy[w] * xv[q][w];
                            a2 += c[q].hz[w] * xv[q][w];
                        }
                }
            }
            a0 = group_sum_t<G>(a0);
            a1 = group_sum_t<G>(a1);
            a2 = group_sum_t<G>(a2);
            if (v < vb && sl == 0) u[v] = V4<T>{a0, a1, a2, (T)0};
        }
        __syncthreads();   // every thread is done with this stage: refill it
        if (t == 0 && jt + VG_STAGES < my_tiles) issue(jt + VG_STAGES);
    }
}

// Eq. 5 position update from the vertex-major gradients: x_v += omega sqrt(w_v) sum_{(j,s) at v}
// h_{j,s} dl_j over the same padded layout (fp64 lane partials, fixed butterfly).
#ifndef MGPBD_UPD_THREADS
#define MGPBD_UPD_THREADS 256
#endif
constexpr int UPD_BS = MGPBD_UPD_THREADS;   // threads per CTA of the Eq. 5 update (build switch)
template <class T, int G, int UN, bool J16>
__global__ void __launch_bounds__(UPD_BS) k_mf_update(int32_t v0, int32_t v1, int64_t npad,
                                                     const int64_t* __restrict__ ppos,
                                                     const uint16_t* __restrict__ vj16,
                                                     const int32_t* __restrict__ vj32,
                                                     const int32_t* __restrict__ jbase, const T* __restrict__ hv,
                                                     const T* __restrict__ dl, const double* __restrict__ sqrtw,
                                                     const double* __restrict__ omega_p, double* __restrict__ x, int nsm) {
    using CH = Chunk<T, J16>;
    constexpr int VW = CH::VW;
    constexpr int PER_WARP = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
    const VRange vr = warp_vertices<PER_WARP>(v0, v1, nsm);  // (the vertex gather's blocked ranges: dl reuse in L1)
    const T* __restrict__ hx = hv;
    const T* __restrict__ hy = hv + npad;
    const T* __restrict__ hz = hv + 2 * npad;
    for (int64_t base = vr.first; base < vr.vend; base += vr.step) {  // warp-uniform
        const int64_t v = base + sub;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if (v < vr.vend) {
            const int64_t p0 = ppos[v], p1 = ppos[v + 1];
            const int32_t jb = J16 ? jbase[v] : 0;
            for (int64_t pb = p0 + (int64_t)sl * VW; pb < p1; pb += (int64_t)G * VW * UN) {
                CH c[UN];
#pragma unroll
                for (int q = 0; q < UN; ++q) {
                    const int64_t p = pb + (int64_t)q * G * VW;
                    c[q].load(hx, hy, hz, vj16, vj32, p, p < p1);
                }
                double dv[UN][VW];
#pragma unroll
                for (int q = 0; q < UN; ++q)
#pragma unroll
                    for (int w = 0; w < VW; ++w) dv[q][w] = (double)dl[jb + c[q].j[w]];
#pragma unroll
                for (int q = 0; q < UN; ++q)
#pragma unroll
                    for (int w = 0; w < VW; ++w) {
                        a0 += (double)c[q].hx[w] * dv[q][w];
                        a1 += (double)c[q].hy[w] * dv[q][w];
                        a2 += (double)c[q].hz[w] * dv[q][w];
                    }
            }
        }
        a0 = group_sum<G>(a0);
        a1 = group_sum<G>(a1);
        a2 = group_sum<G>(a2);
        if (v < vr.vend && sl == 0) {
            const double sw = sqrtw[v], om = *omega_p;
            x[3 * v] += om * (sw * a0);
            x[3 * v + 1] += om * (sw * a1);
            x[3 * v + 2] += om * (sw * a2);
        }
    }
}

// (A x)_i = sum_s h_{i,s} . u_{v_s} + at_i x_i in the storage precision, epilogue in fp64 exactly as
// the CSR row kernels (solve.cu k_rows).
template <class T, int KC, int MODE>
__global__ void __launch_bounds__(MF_BS, 2048 / MF_BS) k_mf_rows(int32_t row0, int32_t row1, const int32_t* __restrict__ verts,
                                                   const T* __restrict__ h, const V4<T>* __restrict__ u,
                                                   const T* __restrict__ at, const T* __restrict__ dinv,
                                                   const T* __restrict__ x, const T* __restrict__ b,
                                                   T* __restrict__ y, const T* __restrict__ aux, double omega,
                                                   double alpha, const T* __restrict__ xprev,
                                                   double* __restrict__ parts, double* __restrict__ parts2) {
    using IV = typename std::conditional<KC == 4, int4, int2>::type;
    double acc1 = 0.0, acc2 = 0.0;
    const int32_t nt = gridDim.x * blockDim.x;
    for (int32_t i = row0 + blockIdx.x * blockDim.x + threadIdx.x; i < row1; i += nt) {
        int vi[KC];
        T hi[KC][3];
        load_iv(reinterpret_cast<const IV*>(verts)[i], vi);
        load_record<T, KC>(h + (int64_t)i * KC * 3, hi);
        const T xi = x[i];
        T acc = at[i] * xi;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const V4<T> uu = u[vi[k]];
            acc += hi[k][0] * uu.x + hi[k][1] * uu.y + hi[k][2] * uu.z;
        }
        const double s = (double)acc;
        if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) {
            double yd = (double)xi + omega * (double)dinv[i] * ((double)b[i] - s);
            if (alpha != 0.0) yd += alpha * ((double)xi - (xprev ? (double)xprev[i] : 0.0));  // Chebyshev step
            const T yi = (T)yd;
            y[i] = yi;
            if (MODE == PASS_JACOBI_DOT) {
                const double ai = (double)aux[i];
                acc1 += ai * (double)yi;
                acc2 += ai * ai;
            }
        } else if (MODE == PASS_RESID_P) {
            y[i] = (T)((double)aux[i] * ((double)b[i] - s));
        } else if (MODE == PASS_SPMV_DOT) {
            const T yi = (T)s;
            y[i] = yi;
            acc1 += (double)xi * (double)yi;
        } else if (MODE == PASS_POWER) {
            const T yi = (T)((double)dinv[i] * s);
            y[i] = yi;
            acc1 += (double)yi * (double)yi;
        }
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        const double t1 = block_sum<MF_BS>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            const double t2 = block_sum<MF_BS>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// TMA-pipelined row kernel: persistent CTAs stream MF_R-row tiles of the constraint records (vertex
// ids, h) and per-row operands into shared memory with 1-D bulk copies (cp.async.bulk, completion on
// an mbarrier), MF_STAGES deep, so the HBM stream never waits on the dependent u gathers.

#ifndef MGPBD_ROWS_PIPE
#define MGPBD_ROWS_PIPE 1
#endif
#ifndef MGPBD_ROWS_TRIGGER
#define MGPBD_ROWS_TRIGGER 0
#endif
#ifndef MGPBD_ROWS_BLOCKED
#define MGPBD_ROWS_BLOCKED 1
#endif
template <class T, int KC, bool V16>
struct TileLayout {  // byte offsets inside one stage (every section 16-B aligned for R = 128 or 256)
    static constexpr int R = mf_r<T, KC>();
    static constexpr uint32_t VB = V16 ? 2 : 4;  // bytes per vertex index (16-bit: offset from the tile's base)
    static constexpr uint32_t H = 0;
    static constexpr uint32_t V = H + R * KC * 3 * sizeof(T);
    static constexpr uint32_t X = V + R * KC * VB;
    static constexpr uint32_t AT = X + R * sizeof(T);
    static constexpr uint32_t D = AT + R * sizeof(T);
    static constexpr uint32_t B = D + R * sizeof(T);
    static constexpr uint32_t AUX = B + R * sizeof(T);
    static constexpr uint32_t XP = AUX + R * sizeof(T);
    static constexpr uint32_t BYTES = XP + R * sizeof(T);
};

template <class T, int KC, int MODE, bool V16>
__global__ void __launch_bounds__(mf_r<T, KC>()) k_mf_rows_tma(int32_t row0, int32_t row1, int32_t tbase, int32_t ntiles,
                                                      const void* __restrict__ verts_, const int32_t* __restrict__ vbase,
                                                      const T* __restrict__ h,
                                                      const V4<T>* __restrict__ u, const T* __restrict__ at,
                                                      const T* __restrict__ dinv, const T* __restrict__ x,
                                                      const T* __restrict__ b, T* __restrict__ y,
                                                      const T* __restrict__ aux, double omega, double alpha,
                                                      const T* __restrict__ xprev, double* __restrict__ parts,
                                                      double* __restrict__ parts2, double xom, double* __restrict__ fin,
                                                      unsigned* __restrict__ fin_ctr) {
    // xom != 0 (PASS_JACOBI only): x is not materialised, x_i = xom D^-1_ii b_i (see k_mf_vgather XJ)
    using LY = TileLayout<T, KC, V16>;
    constexpr int MF_RK = LY::R;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[MF_STAGES];
    constexpr bool ND = MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT || MODE == PASS_POWER;
    constexpr bool NB = MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT || MODE == PASS_RESID_P;
    constexpr bool NA = MODE == PASS_JACOBI_DOT || MODE == PASS_RESID_P;
    const bool NP = (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) && alpha != 0.0 && xprev != nullptr;
    const int t = threadIdx.x;
    if (t == 0) {
        for (int k = 0; k < MF_STAGES; ++k) mbar_init(&bars[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // tile j of this CTA: blockIdx.x + j gridDim.x (round robin), or (MGPBD_ROWS_BLOCKED) blockIdx.x tpc + j over
    // a contiguous range of tpc tiles; rows [tbase + tile R, +R) clipped to row1
    const int tpc = (ntiles + (int)gridDim.x - 1) / (int)gridDim.x;
    auto tile_of = [&](int j) { return MGPBD_ROWS_BLOCKED ? (int)blockIdx.x * tpc + j : (int)blockIdx.x + j * (int)gridDim.x; };
    auto issue = [&](int j) {
        const int tile = tile_of(j);
        unsigned char* st = smem + (size_t)(j % MF_STAGES) * LY::BYTES;
        const int32_t i0 = tbase + tile * MF_RK;
        const int32_t rows = min(MF_RK, row1 - i0);
        auto rnd = [](uint32_t by) { return (by + 15u) & ~15u; };
        const uint32_t bh = rnd(rows * KC * 3 * sizeof(T)), bv = rnd(rows * KC * LY::VB),
                       bs = rnd(rows * sizeof(T));
        const bool XJ = xom != 0.0;
        uint32_t tot = bh + bv + (XJ ? 0 : bs) + bs + (ND ? bs : 0) + (NB ? bs : 0) + (NA ? bs : 0) + (NP ? bs : 0);
        uint64_t* bar = &bars[j % MF_STAGES];
        mbar_expect_tx(bar, tot);
        if constexpr (MGPBD_L2POL == 1 || MGPBD_L2POL == 2) {
            const uint64_t pol = MGPBD_L2POL == 1 ? l2_policy_first() : l2_policy_last();
            bulk_g2s_pol(st + LY::H, h + (int64_t)i0 * KC * 3, bh, bar, pol);
            bulk_g2s_pol(st + LY::V, reinterpret_cast<const unsigned char*>(verts_) + (int64_t)i0 * KC * LY::VB, bv, bar,
                         pol);
        } else {
            bulk_g2s(st + LY::H, h + (int64_t)i0 * KC * 3, bh, bar);
            bulk_g2s(st + LY::V, reinterpret_cast<const unsigned char*>(verts_) + (int64_t)i0 * KC * LY::VB, bv, bar);
        }
        if (!XJ) bulk_g2s(st + LY::X, x + i0, bs, bar);
        bulk_g2s(st + LY::AT, at + i0, bs, bar);
        if (ND) bulk_g2s(st + LY::D, dinv + i0, bs, bar);
        if (NB) bulk_g2s(st + LY::B, b + i0, bs, bar);
        if (NA) bulk_g2s(st + LY::AUX, aux + i0, bs, bar);
        if (NP) bulk_g2s(st + LY::XP, xprev + i0, bs, bar);
    };
    const int my_tiles = MGPBD_ROWS_BLOCKED ? max(0, min(tpc, ntiles - (int)blockIdx.x * tpc))
                                            : (blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
    if (t == 0)
        for (int j = 0; j < MF_STAGES && j < my_tiles; ++j) issue(j);
    // everything above reads only data of earlier kernels; u comes from the vertex gather launched
    // just before this grid (programmatic dependent launch): wait for it before the first gather
    asm volatile("griddepcontrol.wait;" ::: "memory");
    double acc1 = 0.0, acc2 = 0.0;
    // u of tile j is gathered one tile ahead (MGPBD_ROWS_PIPE): while tile j's products run, the L2 round trip of
    // tile j + 1's gathers is in flight (its stage has landed: the ring is MF_STAGES >= 2 deep)
    auto rowof = [&](int j) { return tbase + tile_of(j) * MF_RK + t; };
    auto gather_u = [&](int j, V4<T> (&uo)[KC]) {
        mbar_wait(&bars[j % MF_STAGES], (uint32_t)((j / MF_STAGES) & 1));
        const unsigned char* st = smem + (size_t)(j % MF_STAGES) * LY::BYTES;
        const int32_t i = rowof(j);
        if (i >= row0 && i < row1) {
            int vi[KC];
            if (V16) {
                const uint16_t* sv = reinterpret_cast<const uint16_t*>(st + LY::V) + t * KC;
                const int32_t vb = vbase[tile_of(j)];
#pragma unroll
                for (int k = 0; k < KC; ++k) vi[k] = vb + (int32_t)sv[k];
            } else {
                const int32_t* sv = reinterpret_cast<const int32_t*>(st + LY::V) + t * KC;
#pragma unroll
                for (int k = 0; k < KC; ++k) vi[k] = sv[k];
            }
#pragma unroll
            for (int k = 0; k < KC; ++k) uo[k] = u[vi[k]];
        }
    };
    V4<T> uc[KC];
    if (MGPBD_ROWS_PIPE && my_tiles > 0) gather_u(0, uc);
    for (int j = 0; j < my_tiles; ++j) {
        V4<T> un[KC];
        if (MGPBD_ROWS_PIPE) {
            if (j + 1 < my_tiles) gather_u(j + 1, un);
        } else {
            gather_u(j, uc);
        }
        const unsigned char* st = smem + (size_t)(j % MF_STAGES) * LY::BYTES;
        const int32_t i = rowof(j);
        if (i >= row0 && i < row1) {
            T hi[KC][3];
            load_record<T, KC>(reinterpret_cast<const T*>(st + LY::H) + t * KC * 3, hi);
            const T xi = xom != 0.0 ? (T)(xom * (double)reinterpret_cast<const T*>(st + LY::D)[t] *
                                          (double)reinterpret_cast<const T*>(st + LY::B)[t])
                                    : reinterpret_cast<const T*>(st + LY::X)[t];
            T acc = reinterpret_cast<const T*>(st + LY::AT)[t] * xi;
#pragma unroll
            for (int k = 0; k < KC; ++k) acc += hi[k][0] * uc[k].x + hi[k][1] * uc[k].y + hi[k][2] * uc[k].z;
            const double s = (double)acc;
            const double di = ND ? (double)reinterpret_cast<const T*>(st + LY::D)[t] : 0.0;
            const double bi = NB ? (double)reinterpret_cast<const T*>(st + LY::B)[t] : 0.0;
            const double ai = NA ? (double)reinterpret_cast<const T*>(st + LY::AUX)[t] : 0.0;
            if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) {
                double yd = (double)xi + omega * di * (bi - s);
                if (alpha != 0.0)
                    yd += alpha * ((double)xi - (NP ? (double)reinterpret_cast<const T*>(st + LY::XP)[t] : 0.0));
                const T yi = (T)yd;
                y[i] = yi;
                if (MODE == PASS_JACOBI_DOT) { acc1 += ai * (double)yi; acc2 += ai * ai; }
            } else if (MODE == PASS_RESID_P) {
                y[i] = (T)(ai * (bi - s));
            } else if (MODE == PASS_SPMV_DOT) {
                const T yi = (T)s;
                y[i] = yi;
                acc1 += (double)xi * (double)yi;
            } else if (MODE == PASS_POWER) {
                const T yi = (T)(di * s);
                y[i] = yi;
                acc1 += (double)yi * (double)yi;
            }
        }
        __syncthreads();  // every thread is done with this stage: refill it
        if (t == 0 && j + MF_STAGES < my_tiles) issue(j + MF_STAGES);
        // dependents (the next pass's PDL vertex gather) may launch once this CTA's last tile is done
        // (MGPBD_ROWS_TRIGGER=1; default 0: only at grid completion — the early trigger cost 3 us per back-to-back pass)
        if (MGPBD_ROWS_TRIGGER && j + 1 == my_tiles) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (MGPBD_ROWS_PIPE) {
#pragma unroll
            for (int k = 0; k < KC; ++k) uc[k] = un[k];
        }
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        const double t1 = block_sum<MF_RK>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            const double t2 = block_sum<MF_RK>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
        if ((MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT) && fin) {
            // the last CTA to arrive sums every CTA's partial in index order (deterministic) for the PCG update
            __shared__ int last;
            if (threadIdx.x == 0) {
                __threadfence();
                last = atomicAdd(fin_ctr, 1u) == gridDim.x - 1;
            }
            __syncthreads();
            if (last) {
                __threadfence();
                double a = 0.0, c = 0.0;
                for (int i = threadIdx.x; i < (int)gridDim.x; i += MF_RK) {
                    a += __ldcg(parts + i);
                    if (MODE == PASS_JACOBI_DOT) c += __ldcg(parts2 + i);
                }
                a = block_sum<MF_RK>(a, sh);
                if (MODE == PASS_JACOBI_DOT) c = block_sum<MF_RK>(c, sh);
                if (threadIdx.x == 0) {
                    if (MODE == PASS_JACOBI_DOT) { fin[0] = a; fin[1] = c; }
                    else fin[2] = a;
                    *fin_ctr = 0u;
                }
            }
        }
    }
}

template <class T, int KC>
void mf_pass_kc(int mode, const MatFree<T>& A, const T* x, const T* b, T* y, const T* aux, double omega,
                double* parts, double* parts2, cudaStream_t s, double alpha, const T* xprev, double xom,
                const std::function<void()>* mid) {
    if (xom != 0.0 && (mode != PASS_JACOBI || !A.tma || A.vg_ts > 0))
        throw Error(-1, "mf_pass: implicit x (x0_omega) needs PASS_JACOBI and the TMA row kernel");
    // the vertex gather over [gv0, gv1)
    auto gather = [&](int32_t gv0, int32_t gv1) {
        if (gv1 <= gv0) return;
        // G lanes per vertex, UN 16-byte chunks per lane per round (~23 incidences per vertex on tets = 6 float4
        // chunks, ~6 on cloth = 2); build-time overridable for tuning sweeps
#ifndef MGPBD_VG_G
#define MGPBD_VG_G 4
#endif
#ifndef MGPBD_VG_UN
#define MGPBD_VG_UN 2
#endif
        constexpr int G = KC == 4 ? MGPBD_VG_G : 2;
#ifndef MGPBD_VG_UN64
#define MGPBD_VG_UN64 3
#endif
        // fp64 chunks hold 2 incidences: 3 per lane per round cover a tet vertex (78.6 vs 87.2 us per pass at 2)
        constexpr int UN = KC == 4 ? (sizeof(T) == 8 ? MGPBD_VG_UN64 : MGPBD_VG_UN) : 1;
        const int64_t thr = (int64_t)(gv1 - gv0) * G;
#ifndef MGPBD_VG_CTAS_PER_SM
#define MGPBD_VG_CTAS_PER_SM 16
#endif
        int grid = (int)std::min<int64_t>((thr + vg_threads<T>() - 1) / vg_threads<T>(), 148 * MGPBD_VG_CTAS_PER_SM);
        if (MGPBD_VG_BLOCKED) {  // persistent: the resident CTAs only
            static const int resident = [] {
                int occ = 1;
                MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mf_vgather<T, G, UN, true, false>, vg_threads<T>(), 0));
                return std::max(1, occ);
            }();
            grid = (int)std::min<int64_t>((thr + vg_threads<T>() - 1) / vg_threads<T>(), (int64_t)vg_sms() * resident);
        }
        if (A.vg_grid_cap > 0) grid = std::min(grid, A.vg_grid_cap);
        if (A.vg_ts > 0) {  // TMA-pipelined vertex gather
            constexpr int GT = KC == 4 ? 4 : 2;
            const int32_t ntiles = (gv1 - gv0 + VGT - 1) / VGT;
            int tg = std::min(ntiles, A.vg_grid);
            if (A.vg_grid_cap > 0) tg = std::min(tg, A.vg_grid_cap);
            if (A.vj16) {
                const size_t sm = (size_t)VG_STAGES * VgLayout<T, true>(A.vg_ts).bytes;
                ensure_dyn_smem((const void*)k_mf_vgather_tma<T, GT, true>, sm);
                k_mf_vgather_tma<T, GT, true><<<tg, VG_BS, sm, s>>>(gv0, gv1, ntiles, A.vg_ts, A.npad, A.ppos, A.vj16,
                                                                   A.vj32, A.jbase, A.hv, x, reinterpret_cast<V4<T>*>(A.u));
            } else {
                const size_t sm = (size_t)VG_STAGES * VgLayout<T, false>(A.vg_ts).bytes;
                ensure_dyn_smem((const void*)k_mf_vgather_tma<T, GT, false>, sm);
                k_mf_vgather_tma<T, GT, false><<<tg, VG_BS, sm, s>>>(gv0, gv1, ntiles, A.vg_ts, A.npad, A.ppos, A.vj16,
                                                                    A.vj32, A.jbase, A.hv, x, reinterpret_cast<V4<T>*>(A.u));
            }
        } else {
#define MG_VG(J, X)                                                                                     \
    do {                                                                                                \
        cudaLaunchConfig_t lc = {};                                                                     \
        lc.gridDim = dim3(grid);                                                                        \
        lc.blockDim = dim3(vg_threads<T>());                                                                 \
        lc.stream = s;                                                                                  \
        cudaLaunchAttribute la[1];                                                                      \
        la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                  \
        la[0].val.programmaticStreamSerializationAllowed = 1;                                           \
        lc.attrs = la;                                                                                  \
        lc.numAttrs = A.vg_pdl ? 1 : 0;                                                                 \
        MG_CK(cudaLaunchKernelEx(&lc, k_mf_vgather<T, G, UN, J, X>, gv0, gv1, A.npad, A.ppos, A.vj16, \
                                 A.vj32, A.jbase, A.hv, x, reinterpret_cast<V4<T>*>(A.u), (const T*)A.dinv, \
                                 b, xom, vg_sms()));                                                    \
    } while (0)
            if (A.vj16) { if (xom != 0.0) MG_VG(true, true); else MG_VG(true, false); }
            else { if (xom != 0.0) MG_VG(false, true); else MG_VG(false, false); }
#undef MG_VG
        }
        MG_LAUNCH_CHECK();
    };
    // mid (partitioned level 0, MatFree::vi0/vi1): the interior vertices — no halo incidence — are gathered while the
    // halo exchange runs; mid() joins it, then the boundary vertices
    if (mid && A.vi1 > A.vi0 && A.vg_ts == 0) {
        gather(A.vi0, A.vi1);
        (*mid)();
        gather(A.v0, A.vi0);
        gather(A.vi1, A.v1);
    } else {
        if (mid) (*mid)();
        gather(A.v0, A.v1);
    }
    const V4<T>* u = reinterpret_cast<const V4<T>*>(A.u);
    if (A.tma) {
        const int32_t tbase = A.row0 & ~3;  // 16-B aligned vector offsets
        constexpr int R = mf_r<T, KC>();
        const int32_t ntiles = (A.row1 - tbase + R - 1) / R;
#define MG_MFT(M) { if (A.v16) MG_MFT2(M, true) else MG_MFT2(M, false) }
#define MG_MFT2(M, V16)                                                                                         \
    {                                                                                                           \
        const size_t smem = (size_t)MF_STAGES * TileLayout<T, KC, V16>::BYTES;                                  \
        ensure_dyn_smem((const void*)k_mf_rows_tma<T, KC, M, V16>, smem);                                      \
        cudaLaunchConfig_t lc = {};                                                                             \
        lc.gridDim = dim3(A.grid);                                                                              \
        lc.blockDim = dim3(R);                                                                                  \
        lc.dynamicSmemBytes = smem;                                                                             \
        lc.stream = s;                                                                                          \
        cudaLaunchAttribute la[1];                                                                              \
        la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                          \
        la[0].val.programmaticStreamSerializationAllowed = 1;                                                   \
        lc.attrs = la;                                                                                          \
        lc.numAttrs = 1;                                                                                        \
        MG_CK(cudaLaunchKernelEx(&lc, k_mf_rows_tma<T, KC, M, V16>, A.row0, A.row1, tbase, ntiles,              \
                                 V16 ? (const void*)A.v16 : (const void*)A.verts, A.vbase, A.h, u,              \
                                 (const T*)A.at, (const T*)A.dinv, x, b, y, aux, omega, alpha, xprev, parts,    \
                                 parts2, xom, A.fin, A.fin_ctr));                                               \
    }
        switch (mode) {
            case PASS_JACOBI: MG_MFT(PASS_JACOBI); break;
            case PASS_JACOBI_DOT: MG_MFT(PASS_JACOBI_DOT); break;
            case PASS_RESID_P: MG_MFT(PASS_RESID_P); break;
            case PASS_SPMV_DOT: MG_MFT(PASS_SPMV_DOT); break;
            case PASS_POWER: MG_MFT(PASS_POWER); break;
            default: throw Error(-1, "mf_pass: bad mode");
        }
#undef MG_MFT
#undef MG_MFT2
        MG_LAUNCH_CHECK();
        return;
    }
#define MG_MF(M)                                                                                            \
    k_mf_rows<T, KC, M><<<A.grid, MF_BS, 0, s>>>(A.row0, A.row1, A.verts, A.h, u, A.at, A.dinv, x, b, y, aux, \
                                                  omega, alpha, xprev, parts, parts2)
    switch (mode) {
        case PASS_JACOBI: MG_MF(PASS_JACOBI); break;
        case PASS_JACOBI_DOT: MG_MF(PASS_JACOBI_DOT); break;
        case PASS_RESID_P: MG_MF(PASS_RESID_P); break;
        case PASS_SPMV_DOT: MG_MF(PASS_SPMV_DOT); break;
        case PASS_POWER: MG_MF(PASS_POWER); break;
        default: throw Error(-1, "mf_pass: bad mode");
    }
#undef MG_MF
    MG_LAUNCH_CHECK();
}

}  // namespace

int mf_grid(int32_t rows) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)rows + MF_BS - 1) / MF_BS, 148 * 8));
}

int mf_vg_plan(const std::vector<int64_t>& ppos, int32_t v0, int32_t v1, int tsize, bool j16, int* grid) {
    int64_t ts = 4;
    for (int64_t v = v0; v < v1; v += VGT) ts = std::max<int64_t>(ts, ppos[std::min<int64_t>(v + VGT, v1)] - ppos[v]);
    if (ts > (1 << 20)) return 0;
    const uint32_t bytes = tsize == 4 ? (j16 ? VgLayout<float, true>((int32_t)ts).bytes : VgLayout<float, false>((int32_t)ts).bytes)
                                      : (j16 ? VgLayout<double, true>((int32_t)ts).bytes : VgLayout<double, false>((int32_t)ts).bytes);
    const int per_sm = (int)std::min<size_t>(std::min(16, 2048 / VG_BS), (227 * 1024) / ((size_t)VG_STAGES * bytes + 1024));
    if (per_sm < 1) return 0;
    int dev = 0, sms = 148;
    MG_CK(cudaGetDevice(&dev));
    MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    *grid = sms * per_sm;
    return (int)ts;
}

bool mf_build_v16(int32_t row0, int32_t row1, int kc, int tsize, const std::vector<int32_t>& hverts,
                  DBuf<uint16_t>& v16, DBuf<int32_t>& vbase, cudaStream_t s) {
    const int32_t tbase = row0 & ~3;
    const int R = mf_r(kc, tsize);
    const int64_t ntiles = std::max<int64_t>(1, ((int64_t)row1 - tbase + R - 1) / R);
    const int64_t m = (int64_t)hverts.size() / kc;
    std::vector<int32_t> vb((size_t)ntiles, 0);
    std::vector<uint16_t> o((size_t)m * kc, 0);
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t i0 = tbase + t * R, i1 = std::min<int64_t>(i0 + R, row1);
        int32_t lo = INT32_MAX, hi = -1;
        for (int64_t e = i0 * kc; e < i1 * kc; ++e) { lo = std::min(lo, hverts[e]); hi = std::max(hi, hverts[e]); }
        if (hi < 0) continue;
        if (hi - lo >= 65536) return false;
        vb[t] = lo;
        for (int64_t e = i0 * kc; e < i1 * kc; ++e) o[e] = (uint16_t)(hverts[e] - lo);
    }
    v16.resize((size_t)m * kc);
    h2d(v16.p, o.data(), (size_t)m * kc, s);
    vbase.resize((size_t)ntiles);
    h2d(vbase.p, vb.data(), (size_t)ntiles, s);
    MG_CK(cudaStreamSynchronize(s));
    return true;
}

int mf_grid_tma(int32_t row0, int32_t row1, int tsize, int kc, int vbytes) {
    const int32_t tbase = row0 & ~3;
    const int R = mf_r(kc, tsize);
    const int64_t ntiles = std::max<int64_t>(1, ((int64_t)row1 - tbase + R - 1) / R);
    const size_t stage = (size_t)R * ((size_t)kc * 3 * tsize + (size_t)kc * vbytes + 6 * (size_t)tsize);
#ifndef MGPBD_ROWS_PER_SM
#define MGPBD_ROWS_PER_SM 8
#endif
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(MGPBD_ROWS_PER_SM, (227 * 1024) / (MF_STAGES * stage + 1024)));
    int dev = 0, sms = 148;
    MG_CK(cudaGetDevice(&dev));
    MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
}

template <class T>
void mf_refresh(const MatFree<T>& A, const double* alpha, double dt, T* dinv, cudaStream_t s) {
    const int64_t work = std::max<int64_t>(A.p1 - A.p0, A.m);
    if (work <= 0) return;
    const int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
    if (A.kc == 4)
        k_mf_refresh<T, 4><<<grid, 256, 0, s>>>(A.p0, A.p1, A.npad, A.vsrc, A.h, A.hv, A.m, A.row0, A.row1, alpha,
                                                dt * dt, A.at, dinv);
    else
        k_mf_refresh<T, 2><<<grid, 256, 0, s>>>(A.p0, A.p1, A.npad, A.vsrc, A.h, A.hv, A.m, A.row0, A.row1, alpha,
                                                dt * dt, A.at, dinv);
    MG_LAUNCH_CHECK();
}

template <class T>
void mf_pass(int mode, const MatFree<T>& A, const T* x, const T* b, T* y, const T* aux, double omega,
             double* parts, double* parts2, cudaStream_t s, double alpha, const T* xprev, double xom,
             const std::function<void()>* mid) {
    if (A.kc == 4) mf_pass_kc<T, 4>(mode, A, x, b, y, aux, omega, parts, parts2, s, alpha, xprev, xom, mid);
    else mf_pass_kc<T, 2>(mode, A, x, b, y, aux, omega, parts, parts2, s, alpha, xprev, xom, mid);
}

// grid of the vertex-major update: the resident CTAs only when the ranges are blocked (persistent), else grid-stride
static int update_grid(const void* k, int64_t threads) {
    int grid = (int)std::min<int64_t>((threads + UPD_BS - 1) / UPD_BS, 148 * 16);
    if (MGPBD_VG_BLOCKED) {
        int occ = 1;
        MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, UPD_BS, 0));
        grid = (int)std::min<int64_t>((threads + UPD_BS - 1) / UPD_BS, (int64_t)vg_sms() * std::max(1, occ));
    }
    return std::max(grid, 1);
}

template <class T>
void mf_update(const MatFree<T>& A, const T* dl, const double* sqrtw, const double* omega, double* x, cudaStream_t s) {
    if (A.v1 <= A.v0) return;
    if (A.kc == 4) {  // same lane split as the vertex gather (G = 4, UN = 2: ~60 registers)
        constexpr int G = 4;
        const int grid = update_grid((const void*)k_mf_update<T, G, 2, true>, (int64_t)(A.v1 - A.v0) * G);
        if (A.vj16) k_mf_update<T, G, 2, true><<<grid, UPD_BS, 0, s>>>(A.v0, A.v1, A.npad, A.ppos, A.vj16, A.vj32, A.jbase, A.hv, dl, sqrtw, omega, x, vg_sms());
        else k_mf_update<T, G, 2, false><<<grid, UPD_BS, 0, s>>>(A.v0, A.v1, A.npad, A.ppos, A.vj16, A.vj32, A.jbase, A.hv, dl, sqrtw, omega, x, vg_sms());
    } else {
        constexpr int G = 2;
        const int grid = update_grid((const void*)k_mf_update<T, G, 1, true>, (int64_t)(A.v1 - A.v0) * G);
        if (A.vj16) k_mf_update<T, G, 1, true><<<grid, UPD_BS, 0, s>>>(A.v0, A.v1, A.npad, A.ppos, A.vj16, A.vj32, A.jbase, A.hv, dl, sqrtw, omega, x, vg_sms());
        else k_mf_update<T, G, 1, false><<<grid, UPD_BS, 0, s>>>(A.v0, A.v1, A.npad, A.ppos, A.vj16, A.vj32, A.jbase, A.hv, dl, sqrtw, omega, x, vg_sms());
    }
    MG_LAUNCH_CHECK();
}

#define MG_INST(T)                                                                                           \
    template void mf_update<T>(const MatFree<T>&, const T*, const double*, const double*, double*, cudaStream_t); \
    template void mf_refresh<T>(const MatFree<T>&, const double*, double, T*, cudaStream_t);                     \
    template void mf_pass<T>(int, const MatFree<T>&, const T*, const T*, T*, const T*, double, double*, double*, \
                             cudaStream_t, double, const T*, double, const std::function<void()>*);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
