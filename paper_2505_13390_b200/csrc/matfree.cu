// Matrix-free level-0 operator, see matfree.cuh.
#include <algorithm>
#include <vector>

#include "matfree.cuh"
#include "tma.cuh"
#include "util.cuh"
#include "record.cuh"
#include "solve.cuh"

namespace mgpbd {

namespace {

constexpr int MF_BS = 256;

template <class T>
struct alignas(4 * sizeof(T)) V4 {
    T x, y, z, w;
};

// hv[plane][e] = h[vlist[e]][plane] for the incidences of vertices [v0, v1); at_i = alpha_i / dt^2 for
// all rows; dinv_i = 1 / (sum_s |h_{i,s}|^2 + at_i) for rows [r0, r1) — the assembly's diagonal formula
// (mesh.cu k_assemble), so the smoother does not need the assembled matrix.
template <class T, int KC>
__global__ void k_mf_refresh(int64_t e0, int64_t e1, int64_t ninc, const int32_t* __restrict__ vlist,
                             const T* __restrict__ h, T* __restrict__ hv, int32_t m, int32_t r0, int32_t r1,
                             const double* __restrict__ alpha, double dt2, T* __restrict__ at,
                             T* __restrict__ dinv) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = e0 + tid; e < e1; e += nt) {
        const T* p = h + (int64_t)vlist[e] * 3;
        hv[e] = p[0];
        hv[ninc + e] = p[1];
        hv[2 * ninc + e] = p[2];
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

// u_v = sum over v's incidences of h_{j,s} x_j: G lanes per vertex, lane partials in incidence order
// strided by G, fixed butterfly (deterministic).
template <class T, int KC, int G>
__global__ void __launch_bounds__(MF_BS) k_mf_vgather(int32_t v0, int32_t v1, int64_t ninc,
                                                      const int64_t* __restrict__ vptr,
                                                      const int32_t* __restrict__ vlist, const T* __restrict__ hv,
                                                      const T* __restrict__ x, V4<T>* __restrict__ u) {
    // programmatic dependent launch: the row kernel may start streaming its static operands now; it
    // waits (griddepcontrol.wait) for this grid's u before gathering it
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    constexpr int PER_WARP = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T* __restrict__ hx = hv;
    const T* __restrict__ hy = hv + ninc;
    const T* __restrict__ hz = hv + 2 * ninc;
    // warp-uniform trip count: the butterfly below needs the whole warp
    for (int64_t base = v0 + warp * PER_WARP; base < v1; base += nwarps * PER_WARP) {
        const int64_t v = base + sub;
        T a0 = (T)0, a1 = (T)0, a2 = (T)0;
        if (v < v1) {
            // chunks of UN incidences per lane: all index/h loads, then all x gathers, then the FMAs,
            // so a chunk costs two dependent round trips instead of two per incidence
#ifndef MGPBD_VG_UN
#define MGPBD_VG_UN 6  // swept on B200 (profiles/r1/sweep_level0_pass.txt): 6 > 4 > 8 > 2
#endif
            constexpr int UN = MGPBD_VG_UN;
            const int64_t e0 = vptr[v], e1 = vptr[v + 1];
            for (int64_t eb = e0 + sl; eb < e1; eb += G * UN) {
                int32_t cj[UN];
                T px[UN], py[UN], pz[UN], xv[UN];
#pragma unroll
                for (int q = 0; q < UN; ++q) {
                    const int64_t e = eb + q * G;
                    const bool in = e < e1;
                    cj[q] = in ? vlist[e] / KC : -1;
                    px[q] = in ? hx[e] : (T)0;
                    py[q] = in ? hy[e] : (T)0;
                    pz[q] = in ? hz[e] : (T)0;
                }
#pragma unroll
                for (int q = 0; q < UN; ++q) xv[q] = cj[q] >= 0 ? x[cj[q]] : (T)0;
#pragma unroll
                for (int q = 0; q < UN; ++q) {
                    a0 += px[q] * xv[q];
                    a1 += py[q] * xv[q];
                    a2 += pz[q] * xv[q];
                }
            }
        }
        a0 = group_sum_t<G>(a0);
        a1 = group_sum_t<G>(a1);
        a2 = group_sum_t<G>(a2);
        if (v < v1 && sl == 0) u[v] = V4<T>{a0, a1, a2, (T)0};
    }
}

// Eq. 5 position update from the vertex-major gradients: x_v += omega sqrt(w_v) sum_{(j,s) at v}
// h_{j,s} dl_j, G lanes per vertex over the vertex's contiguous incidences in hv (coalesced planes
// instead of one scattered 12-byte record per incidence), fp64 lane partials, fixed butterfly.
template <class T, int KC, int G>
__global__ void __launch_bounds__(MF_BS) k_mf_update(int32_t v0, int32_t v1, int64_t ninc,
                                                     const int64_t* __restrict__ vptr,
                                                     const int32_t* __restrict__ vlist, const T* __restrict__ hv,
                                                     const T* __restrict__ dl, const double* __restrict__ sqrtw,
                                                     const double* __restrict__ omega_p, double* __restrict__ x) {
    constexpr int PER_WARP = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T* __restrict__ hx = hv;
    const T* __restrict__ hy = hv + ninc;
    const T* __restrict__ hz = hv + 2 * ninc;
    for (int64_t base = v0 + warp * PER_WARP; base < v1; base += nwarps * PER_WARP) {  // warp-uniform
        const int64_t v = base + sub;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if (v < v1) {
            constexpr int UN = 4;
            const int64_t e0 = vptr[v], e1 = vptr[v + 1];
            for (int64_t eb = e0 + sl; eb < e1; eb += G * UN) {
                int32_t cj[UN];
                T px[UN], py[UN], pz[UN];
                double dv[UN];
#pragma unroll
                for (int q = 0; q < UN; ++q) {
                    const int64_t e = eb + q * G;
                    const bool in = e < e1;
                    cj[q] = in ? vlist[e] / KC : -1;
                    px[q] = in ? hx[e] : (T)0;
                    py[q] = in ? hy[e] : (T)0;
                    pz[q] = in ? hz[e] : (T)0;
                }
#pragma unroll
                for (int q = 0; q < UN; ++q) dv[q] = cj[q] >= 0 ? (double)dl[cj[q]] : 0.0;
#pragma unroll
                for (int q = 0; q < UN; ++q) {
                    a0 += (double)px[q] * dv[q];
                    a1 += (double)py[q] * dv[q];
                    a2 += (double)pz[q] * dv[q];
                }
            }
        }
        a0 = group_sum<G>(a0);
        a1 = group_sum<G>(a1);
        a2 = group_sum<G>(a2);
        if (v < v1 && sl == 0) {
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
#ifndef MGPBD_MF_R
#define MGPBD_MF_R 128  // swept on B200 (profiles/r1/sweep_level0_pass.txt): 128 rows, 3 stages, 6 CTAs/SM
#endif
constexpr int MF_R = MGPBD_MF_R;  // rows per tile (= threads per CTA)
#ifndef MGPBD_MF_STAGES
#define MGPBD_MF_STAGES 3
#endif
constexpr int MF_STAGES = MGPBD_MF_STAGES;  // ring depth (overridable at build time for tuning sweeps)

template <class T, int KC>
struct TileLayout {  // byte offsets inside one stage (every section 16-B aligned for MF_R = 128 or 256)
    static constexpr uint32_t H = 0;
    static constexpr uint32_t V = H + MF_R * KC * 3 * sizeof(T);
    static constexpr uint32_t X = V + MF_R * KC * sizeof(int32_t);
    static constexpr uint32_t AT = X + MF_R * sizeof(T);
    static constexpr uint32_t D = AT + MF_R * sizeof(T);
    static constexpr uint32_t B = D + MF_R * sizeof(T);
    static constexpr uint32_t AUX = B + MF_R * sizeof(T);
    static constexpr uint32_t XP = AUX + MF_R * sizeof(T);
    static constexpr uint32_t BYTES = XP + MF_R * sizeof(T);
};

template <class T, int KC, int MODE>
__global__ void __launch_bounds__(MF_R) k_mf_rows_tma(int32_t row0, int32_t row1, int32_t tbase, int32_t ntiles,
                                                      const int32_t* __restrict__ verts, const T* __restrict__ h,
                                                      const V4<T>* __restrict__ u, const T* __restrict__ at,
                                                      const T* __restrict__ dinv, const T* __restrict__ x,
                                                      const T* __restrict__ b, T* __restrict__ y,
                                                      const T* __restrict__ aux, double omega, double alpha,
                                                      const T* __restrict__ xprev, double* __restrict__ parts,
                                                      double* __restrict__ parts2) {
    using LY = TileLayout<T, KC>;
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
    // tile j of this CTA = blockIdx.x + j * gridDim.x; rows [tbase + tile*R, +R) clipped to row1
    auto issue = [&](int j) {
        const int tile = blockIdx.x + j * gridDim.x;
        unsigned char* st = smem + (size_t)(j % MF_STAGES) * LY::BYTES;
        const int32_t i0 = tbase + tile * MF_R;
        const int32_t rows = min(MF_R, row1 - i0);
        auto rnd = [](uint32_t by) { return (by + 15u) & ~15u; };
        const uint32_t bh = rnd(rows * KC * 3 * sizeof(T)), bv = rnd(rows * KC * sizeof(int32_t)),
                       bs = rnd(rows * sizeof(T));
        uint32_t tot = bh + bv + 2 * bs + (ND ? bs : 0) + (NB ? bs : 0) + (NA ? bs : 0) + (NP ? bs : 0);
        uint64_t* bar = &bars[j % MF_STAGES];
        mbar_expect_tx(bar, tot);
        bulk_g2s(st + LY::H, h + (int64_t)i0 * KC * 3, bh, bar);
        bulk_g2s(st + LY::V, verts + (int64_t)i0 * KC, bv, bar);
        bulk_g2s(st + LY::X, x + i0, bs, bar);
        bulk_g2s(st + LY::AT, at + i0, bs, bar);
        if (ND) bulk_g2s(st + LY::D, dinv + i0, bs, bar);
        if (NB) bulk_g2s(st + LY::B, b + i0, bs, bar);
        if (NA) bulk_g2s(st + LY::AUX, aux + i0, bs, bar);
        if (NP) bulk_g2s(st + LY::XP, xprev + i0, bs, bar);
    };
    const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (t == 0)
        for (int j = 0; j < MF_STAGES && j < my_tiles; ++j) issue(j);
    // everything above reads only data of earlier kernels; u comes from the vertex gather launched
    // just before this grid (programmatic dependent launch): wait for it before the first gather
    asm volatile("griddepcontrol.wait;" ::: "memory");
    double acc1 = 0.0, acc2 = 0.0;
    for (int j = 0; j < my_tiles; ++j) {
        mbar_wait(&bars[j % MF_STAGES], (uint32_t)((j / MF_STAGES) & 1));
        const unsigned char* st = smem + (size_t)(j % MF_STAGES) * LY::BYTES;
        const int32_t i = tbase + (blockIdx.x + j * gridDim.x) * MF_R + t;
        if (i >= row0 && i < row1) {
            int vi[KC];
            T hi[KC][3];
            {
                const int32_t* sv = reinterpret_cast<const int32_t*>(st + LY::V) + t * KC;
#pragma unroll
                for (int k = 0; k < KC; ++k) vi[k] = sv[k];
                load_record<T, KC>(reinterpret_cast<const T*>(st + LY::H) + t * KC * 3, hi);
            }
            const T xi = reinterpret_cast<const T*>(st + LY::X)[t];
            T acc = reinterpret_cast<const T*>(st + LY::AT)[t] * xi;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const V4<T> uu = u[vi[k]];
                acc += hi[k][0] * uu.x + hi[k][1] * uu.y + hi[k][2] * uu.z;
            }
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
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        const double t1 = block_sum<MF_R>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            const double t2 = block_sum<MF_R>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
    }
}

template <class T, int KC>
void mf_pass_kc(int mode, const MatFree<T>& A, const T* x, const T* b, T* y, const T* aux, double omega,
                double* parts, double* parts2, cudaStream_t s, double alpha, const T* xprev) {
    if (A.v1 > A.v0) {
#ifndef MGPBD_VG_G4
#define MGPBD_VG_G4 4
#endif
        constexpr int G = KC == 4 ? MGPBD_VG_G4 : 2;  // ~23 (tets) / ~6 (cloth) incidences per vertex
        const int64_t thr = (int64_t)(A.v1 - A.v0) * G;
#ifndef MGPBD_VG_CTAS_PER_SM
#define MGPBD_VG_CTAS_PER_SM 16
#endif
        int grid = (int)std::min<int64_t>((thr + MF_BS - 1) / MF_BS, 148 * MGPBD_VG_CTAS_PER_SM);
        if (A.vg_grid_cap > 0) grid = std::min(grid, A.vg_grid_cap);
        k_mf_vgather<T, KC, G><<<grid, MF_BS, 0, s>>>(A.v0, A.v1, A.ninc, A.vptr, A.vlist, A.hv, x,
                                                      reinterpret_cast<V4<T>*>(A.u));
        MG_LAUNCH_CHECK();
    }
    const V4<T>* u = reinterpret_cast<const V4<T>*>(A.u);
    if (A.tma) {
        const int32_t tbase = A.row0 & ~3;  // 16-B aligned vector offsets
        const int32_t ntiles = (A.row1 - tbase + MF_R - 1) / MF_R;
        const size_t smem = (size_t)MF_STAGES * TileLayout<T, KC>::BYTES;
#define MG_MFT(M)                                                                                               \
    {                                                                                                           \
        ensure_dyn_smem((const void*)k_mf_rows_tma<T, KC, M>, smem);                                           \
        cudaLaunchConfig_t lc = {};                                                                             \
        lc.gridDim = dim3(A.grid);                                                                              \
        lc.blockDim = dim3(MF_R);                                                                               \
        lc.dynamicSmemBytes = smem;                                                                             \
        lc.stream = s;                                                                                          \
        cudaLaunchAttribute la[1];                                                                              \
        la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                          \
        la[0].val.programmaticStreamSerializationAllowed = 1;                                                   \
        lc.attrs = la;                                                                                          \
        lc.numAttrs = 1;                                                                                        \
        MG_CK(cudaLaunchKernelEx(&lc, k_mf_rows_tma<T, KC, M>, A.row0, A.row1, tbase, ntiles, A.verts, A.h, u,   \
                                 (const T*)A.at, (const T*)A.dinv, x, b, y, aux, omega, alpha, xprev, parts,    \
                                 parts2));                                                                      \
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

int mf_grid_tma(int32_t row0, int32_t row1, int tsize, int kc) {
    const int32_t tbase = row0 & ~3;
    const int64_t ntiles = std::max<int64_t>(1, ((int64_t)row1 - tbase + MF_R - 1) / MF_R);
    const size_t stage = (size_t)MF_R * ((size_t)kc * 3 * tsize + (size_t)kc * 4 + 6 * (size_t)tsize);
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (227 * 1024) / (MF_STAGES * stage + 1024)));
    int dev = 0, sms = 148;
    MG_CK(cudaGetDevice(&dev));
    MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
}

template <class T>
void mf_refresh(const MatFree<T>& A, const double* alpha, double dt, T* dinv, cudaStream_t s) {
    const int64_t work = std::max<int64_t>(A.e1 - A.e0, A.m);
    if (work <= 0) return;
    const int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
    if (A.kc == 4)
        k_mf_refresh<T, 4><<<grid, 256, 0, s>>>(A.e0, A.e1, A.ninc, A.vlist, A.h, A.hv, A.m, A.row0, A.row1, alpha,
                                                dt * dt, A.at, dinv);
    else
        k_mf_refresh<T, 2><<<grid, 256, 0, s>>>(A.e0, A.e1, A.ninc, A.vlist, A.h, A.hv, A.m, A.row0, A.row1, alpha,
                                                dt * dt, A.at, dinv);
    MG_LAUNCH_CHECK();
}

template <class T>
void mf_pass(int mode, const MatFree<T>& A, const T* x, const T* b, T* y, const T* aux, double omega,
             double* parts, double* parts2, cudaStream_t s, double alpha, const T* xprev) {
    if (A.kc == 4) mf_pass_kc<T, 4>(mode, A, x, b, y, aux, omega, parts, parts2, s, alpha, xprev);
    else mf_pass_kc<T, 2>(mode, A, x, b, y, aux, omega, parts, parts2, s, alpha, xprev);
}

template <class T>
void mf_update(const MatFree<T>& A, const T* dl, const double* sqrtw, const double* omega, double* x, cudaStream_t s) {
    if (A.v1 <= A.v0) return;
    constexpr int G = 4;
    const int64_t thr = (int64_t)(A.v1 - A.v0) * G;
    const int grid = (int)std::min<int64_t>((thr + MF_BS - 1) / MF_BS, 148 * 16);
    if (A.kc == 4)
        k_mf_update<T, 4, G><<<grid, MF_BS, 0, s>>>(A.v0, A.v1, A.ninc, A.vptr, A.vlist, A.hv, dl, sqrtw, omega, x);
    else
        k_mf_update<T, 2, G><<<grid, MF_BS, 0, s>>>(A.v0, A.v1, A.ninc, A.vptr, A.vlist, A.hv, dl, sqrtw, omega, x);
    MG_LAUNCH_CHECK();
}

#define MG_INST(T)                                                                                           \
    template void mf_update<T>(const MatFree<T>&, const T*, const double*, const double*, double*, cudaStream_t); \
    template void mf_refresh<T>(const MatFree<T>&, const double*, double, T*, cudaStream_t);                     \
    template void mf_pass<T>(int, const MatFree<T>&, const T*, const T*, T*, const T*, double, double*, double*, \
                             cudaStream_t, double, const T*);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
