// Hot-loop kernels of the MGPCG solve (see solve.cuh).
#include "solve.cuh"

#include <cooperative_groups.h>
#include <cstdlib>
#include <string>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "util.cuh"

namespace cg = cooperative_groups;

namespace mgpbd {
namespace {

// Relaxation step of the smoother passes: y_i = x_i + omega D^-1 (b - A x)_i, plus the Chebyshev
// momentum alpha (x_i - xprev_i) (xprev == nullptr: xprev = 0).  alpha = 0 is plain omega-Jacobi,
// bit-identical to x_i + omega d_i (b_i - s).
template <class T>
__device__ __forceinline__ double relax(double xi, int64_t i, double omega, double alpha, const T* __restrict__ xprev,
                                        double di, double bi, double s) {
    double y = xi + omega * di * (bi - s);
    if (alpha != 0.0) y += alpha * (xi - (xprev ? (double)xprev[i] : 0.0));
    return y;
}

constexpr int PB = 256;  // threads per block of the CSR passes

inline int vgrid(int64_t n) {
    int64_t g = (n + PB - 1) / PB;
    return (int)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

// One fused pass over a CSR matrix, VL lanes per row, grid-stride over rows with a warp-uniform loop
// (so the fixed-order sub-warp butterfly is always executed by full warps).
template <class T, int VL, int MODE>
__global__ void __launch_bounds__(PB) k_pass(int32_t row0, int32_t n, const int64_t* __restrict__ rowptr,
                                             const int32_t* __restrict__ col, const T* __restrict__ val,
                                             const T* __restrict__ dinv, const T* __restrict__ x,
                                             const T* __restrict__ b, T* __restrict__ y,
                                             const T* __restrict__ aux, double omega, double alpha, const T* __restrict__ xprev, double* __restrict__ parts,
                                             double* __restrict__ parts2) {
    constexpr int RPW = 32 / VL;  // rows per warp
    const int lane = threadIdx.x & 31;
    const int sub = lane % VL, rid = lane / VL;
    const int64_t gw = ((int64_t)blockIdx.x * PB + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * PB) >> 5;
    double acc1 = 0.0, acc2 = 0.0;
    for (int64_t r0 = row0 + gw * RPW; r0 < n; r0 += nw * RPW) {  // rows [row0, n)
        const int64_t i = r0 + rid;
        const bool valid = i < n;
        double s = 0.0;
        if (valid) {
            const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
#pragma unroll 4
            for (int64_t e = e0 + sub; e < e1; e += VL) s += (double)val[e] * (double)x[col[e]];
        }
        s = group_sum<VL>(s);
        if (valid && sub == 0) {
            if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) {
                T yi = (T)relax((double)x[i], i, omega, alpha, xprev, (double)dinv[i], (double)b[i], s);
                y[i] = yi;
                if (MODE == PASS_JACOBI_DOT) {
                    double r = (double)aux[i];
                    acc1 += r * (double)yi;
                    acc2 += r * r;
                }
            } else if (MODE == PASS_RESID_P) {
                y[i] = (T)((double)aux[i] * ((double)b[i] - s));
            } else if (MODE == PASS_SPMV_DOT) {
                T yi = (T)s;
                y[i] = yi;
                acc1 += (double)x[i] * (double)yi;
            } else if (MODE == PASS_POWER) {
                T yi = (T)((double)dinv[i] * s);
                y[i] = yi;
                acc1 += (double)yi * (double)yi;
            }
        }
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        double t1 = block_sum<PB>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            double t2 = block_sum<PB>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
    }
}

// Row-tile CSR pass: a CTA takes R = 256/VLR consecutive rows (a contiguous nnz range), streams
// val/col/x[col] for the whole tile with coalesced, independent loads (many in flight per thread),
// keeps the fp64 products in shared memory, then VLR lanes per row reduce them in fixed order.
template <class T, int VLR, int MODE>
__global__ void __launch_bounds__(PB) k_tile(int32_t row0, int32_t n, const int64_t* __restrict__ rowptr,
                                             const int32_t* __restrict__ col, const T* __restrict__ val,
                                             const T* __restrict__ dinv, const T* __restrict__ x,
                                             const T* __restrict__ b, T* __restrict__ y,
                                             const T* __restrict__ aux, double omega, double alpha, const T* __restrict__ xprev, double* __restrict__ parts,
                                             double* __restrict__ parts2) {
    extern __shared__ double prod[];
    constexpr int R = PB / VLR;
    const int rr = threadIdx.x / VLR, ln = threadIdx.x % VLR;
    const int64_t ntiles = ((int64_t)n - row0 + R - 1) / R;  // rows [row0, n)
    double acc1 = 0.0, acc2 = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = row0 + tile * R;
        const int64_t r1 = r0 + R < n ? r0 + R : n;
        const int64_t e0 = rowptr[r0];
        const int ne = (int)(rowptr[r1] - e0);
        const T* __restrict__ vt = val + e0;
        const int32_t* __restrict__ ct = col + e0;
#pragma unroll 4
        for (int k = threadIdx.x; k < ne; k += PB) prod[k] = (double)vt[k] * (double)x[ct[k]];
        __syncthreads();
        const int64_t i = r0 + rr;
        double s = 0.0;
        if (i < r1) {
            const int a = (int)(rowptr[i] - e0), z = (int)(rowptr[i + 1] - e0);
            for (int k = a + ln; k < z; k += VLR) s += prod[k];
        }
        s = group_sum<VLR>(s);
        if (ln == 0 && i < r1) {
            if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) {
                T yi = (T)relax((double)x[i], i, omega, alpha, xprev, (double)dinv[i], (double)b[i], s);
                y[i] = yi;
                if (MODE == PASS_JACOBI_DOT) {
                    double r = (double)aux[i];
                    acc1 += r * (double)yi;
                    acc2 += r * r;
                }
            } else if (MODE == PASS_RESID_P) {
                y[i] = (T)((double)aux[i] * ((double)b[i] - s));
            } else if (MODE == PASS_SPMV_DOT) {
                T yi = (T)s;
                y[i] = yi;
                acc1 += (double)x[i] * (double)yi;
            } else if (MODE == PASS_POWER) {
                T yi = (T)((double)dinv[i] * s);
                y[i] = yi;
                acc1 += (double)yi * (double)yi;
            }
        }
        __syncthreads();
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        double t1 = block_sum<PB>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            double t2 = block_sum<PB>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
    }
}

// Band-staged row-tile pass (level 0 of mesh-ordered matrices).  One 1024-thread CTA per SM walks
// "band tiles" of C consecutive rows; for each it stages the window x[lo, lo+len) that those rows
// touch into shared memory (one coalesced copy), then processes sub-tiles of 1024/VLR rows: stream
// val/col with independent coalesced loads, gather x from the shared window (no L1 line fan-out),
// products (PT = T) into shared memory, fixed-order VLR-lane row reductions.  The epilogue's per-row
// loads are issued before the stream so their latency overlaps it.
constexpr int BB = 1024;
constexpr int BAND_EPT = 12;  // stream elements per thread per sub-tile (sub-tile nnz + 6 <= BAND_EPT*BB)
template <class T, int VLR, int MODE>
__global__ void __launch_bounds__(BB, 1) k_band(int32_t row0, int32_t n, int32_t C, const int32_t* __restrict__ win_lo,
                                                const int32_t* __restrict__ win_len, int prod_cap,
                                                const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                const T* __restrict__ val, const T* __restrict__ dinv,
                                                const T* __restrict__ x, const T* __restrict__ b, T* __restrict__ y,
                                                const T* __restrict__ aux, double omega, double alpha, const T* __restrict__ xprev, double* __restrict__ parts,
                                                double* __restrict__ parts2) {
    extern __shared__ __align__(16) unsigned char smraw[];
    T* prod = reinterpret_cast<T*>(smraw);
    T* xs = prod + prod_cap + 8;  // prod holds up to 3 leading + 3 trailing vector lanes beyond the tile
    constexpr int R = BB / VLR;
    const int rr = threadIdx.x / VLR, ln = threadIdx.x % VLR;
    const int32_t nband = (n - row0 + C - 1) / C;  // rows [row0, n)
    double acc1 = 0.0, acc2 = 0.0;
    for (int32_t bt = blockIdx.x; bt < nband; bt += gridDim.x) {
        const int32_t lo = win_lo[bt], len = win_len[bt];
        const int32_t c0 = row0 + bt * C, c1 = c0 + C < n ? c0 + C : n;
        __syncthreads();
        for (int32_t k = threadIdx.x; k < len; k += BB) xs[k] = x[lo + k];
        __syncthreads();
        // software pipeline: the next sub-tile's stream and row operands are loaded into registers
        // while the current sub-tile is reduced (one CTA per SM, so nothing else hides the latency)
        // the stream is read as 16-byte vectors of 4 elements from the 4-aligned start below e0
        constexpr int NV = BAND_EPT / 4;
        using V4 = typename std::conditional<sizeof(T) == 4, float4, double4>::type;
        V4 pv[NV];
        int4 pc[NV];
        int32_t nr0 = c0, nr1 = 0;
        int64_t ne0 = 0, nra = 0, nrz = 0, na0 = 0;
        int nne = 0;
        double nbi = 0.0, ndi = 0.0, nai = 0.0;
        auto fetch = [&](int32_t r0) {
            nr0 = r0;
            nr1 = r0 + R < c1 ? r0 + R : c1;
            ne0 = rowptr[r0];
            nne = (int)(rowptr[nr1] - ne0);
            na0 = ne0 & ~(int64_t)3;
            const int nvec = (int)((ne0 + nne - na0 + 3) >> 2);
            const V4* v4 = reinterpret_cast<const V4*>(val + na0);
            const int4* c4 = reinterpret_cast<const int4*>(col + na0);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int q = threadIdx.x + j * BB;
                if (q < nvec) { pv[j] = v4[q]; pc[j] = c4[q]; }
            }
            const int32_t i = r0 + rr;
            if (i < nr1) {
                nra = rowptr[i];
                nrz = rowptr[i + 1];
                if (ln == 0) {
                    if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT || MODE == PASS_RESID_P) nbi = (double)b[i];
                    if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT || MODE == PASS_POWER) ndi = (double)dinv[i];
                    if (MODE == PASS_JACOBI_DOT || MODE == PASS_RESID_P) nai = (double)aux[i];
                }
            }
        };
        fetch(c0);
        while (nr0 < c1) {
            const int32_t r0 = nr0, r1 = nr1;
            const int64_t e0 = ne0, ra = nra, rz = nrz;
            const int ne = nne;
            const int off = (int)(e0 - na0);  // 0..3 leading elements of the first vector outside the tile
            const double bi = nbi, di = ndi, ai = nai;
            const int32_t i = r0 + rr;
            const bool own = i < r1;
            const int nvec = (ne + off + 3) >> 2;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int q = threadIdx.x + j * BB;
                if (q < nvec) {
                    // products in the storage precision T (fp32 variant: FMUL, no conversions); prod is
                    // indexed from the aligned start so each thread writes one 16-byte vector.  Elements
                    // outside [e0, e0+ne) are gathered at a clamped column and never read back.
                    const int32_t c0x = min(max(pc[j].x - lo, 0), len - 1), c0y = min(max(pc[j].y - lo, 0), len - 1);
                    const int32_t c0z = min(max(pc[j].z - lo, 0), len - 1), c0w = min(max(pc[j].w - lo, 0), len - 1);
                    V4 pr;
                    pr.x = pv[j].x * xs[c0x];
                    pr.y = pv[j].y * xs[c0y];
                    pr.z = pv[j].z * xs[c0z];
                    pr.w = pv[j].w * xs[c0w];
                    reinterpret_cast<V4*>(prod)[q] = pr;
                }
            }
            if (r0 + R < c1) fetch(r0 + R);
            else nr0 = c1;
            __syncthreads();
            T sl = (T)0;  // per-lane partial in T, the cross-lane sum in fp64
            if (own)
                for (int k = (int)(ra - e0) + off + ln; k < (int)(rz - e0) + off; k += VLR) sl += prod[k];
            double s = group_sum<VLR>((double)sl);
            if (own && ln == 0) {
                if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) {
                    T yi = (T)relax((double)xs[i - lo], i, omega, alpha, xprev, di, bi, s);
                    y[i] = yi;
                    if (MODE == PASS_JACOBI_DOT) { acc1 += ai * (double)yi; acc2 += ai * ai; }
                } else if (MODE == PASS_RESID_P) {
                    y[i] = (T)(ai * (bi - s));
                } else if (MODE == PASS_SPMV_DOT) {
                    T yi = (T)s;
                    y[i] = yi;
                    acc1 += (double)xs[i - lo] * (double)yi;
                } else if (MODE == PASS_POWER) {
                    T yi = (T)(di * s);
                    y[i] = yi;
                    acc1 += (double)yi * (double)yi;
                }
            }
            __syncthreads();
        }
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        double t1 = block_sum<BB>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            double t2 = block_sum<BB>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
    }
}

// Band-staged row pass without block barriers: after the shared x window of a band tile is staged,
// every VL-lane group owns rows (warp-uniform stepping so the fixed-order butterfly always runs on
// full warps) and keeps the NEXT row's val/col chunks and per-row operands in flight in registers
// while it reduces the current one.  Rows have at most ROWCH*VL entries (checked at configuration).
constexpr int ROWCH = 5;
// col16[e] = col[e] - win_lo[band tile of the row]: the hot copy of the level-0 column indices.
__global__ void k_col16(int32_t row0, int32_t n, int32_t C, const int64_t* __restrict__ rowptr,
                        const int32_t* __restrict__ col, const int32_t* __restrict__ win_lo,
                        uint16_t* __restrict__ col16) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t li = w0; li < n; li += nw) {
        const int64_t i = row0 + li;
        const int32_t lo = win_lo[li / C];
        for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) col16[e] = (uint16_t)(col[e] - lo);
    }
}

template <class T, int VL, int MODE>
__global__ void __launch_bounds__(BB, 1) k_rows(int32_t row0, int32_t n, int32_t C, const int32_t* __restrict__ win_lo,
                                                const int32_t* __restrict__ win_len,
                                                const int64_t* __restrict__ rowptr, const uint16_t* __restrict__ col,
                                                const T* __restrict__ val, const T* __restrict__ dinv,
                                                const T* __restrict__ x, const T* __restrict__ b, T* __restrict__ y,
                                                const T* __restrict__ aux, double omega, double alpha, const T* __restrict__ xprev, double* __restrict__ parts,
                                                double* __restrict__ parts2) {
    extern __shared__ __align__(16) unsigned char smraw[];
    // shared: [row offsets of the band tile, int32 relative to its first nonzero]
    //         [per-row operands b, dinv, aux of the band tile (storage precision)] [x window]
    int32_t* rp = reinterpret_cast<int32_t*>(smraw);
    T* ob = reinterpret_cast<T*>(smraw + (((size_t)(C + 1) * sizeof(int32_t) + 15) & ~(size_t)15));
    T* od = ob + C;
    T* oa = od + C;
    T* xs = oa + C;
    constexpr int SPW = 32 / VL;              // row groups per warp
    constexpr int NSLOT = (BB / 32) * SPW;    // rows in flight per CTA step
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / VL, sl = lane % VL;
    const int32_t nband = (n - row0 + C - 1) / C;  // rows [row0, n)
    double acc1 = 0.0, acc2 = 0.0;
    struct Row {
        int32_t i;
        int len;
        T v[ROWCH];
        uint16_t c[ROWCH];  // window-relative column
    };
    constexpr bool NB = MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT || MODE == PASS_RESID_P;
    constexpr bool ND = MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT || MODE == PASS_POWER;
    constexpr bool NA = MODE == PASS_JACOBI_DOT || MODE == PASS_RESID_P;
    for (int32_t bt = blockIdx.x; bt < nband; bt += gridDim.x) {
        const int32_t lo = win_lo[bt], len = win_len[bt];
        const int32_t c0 = row0 + bt * C, c1 = c0 + C < n ? c0 + C : n;
        const int64_t ebase = rowptr[c0];
        __syncthreads();
        for (int32_t k = threadIdx.x; k < len; k += BB) xs[k] = x[lo + k];
        for (int32_t k = threadIdx.x; k <= c1 - c0; k += BB) rp[k] = (int32_t)(rowptr[c0 + k] - ebase);
        for (int32_t k = threadIdx.x; k < c1 - c0; k += BB) {
            if (NB) ob[k] = b[c0 + k];
            if (ND) od[k] = dinv[c0 + k];
            if (NA) oa[k] = aux[c0 + k];
        }
        __syncthreads();
        const T* __restrict__ vb = val + ebase;
        const uint16_t* __restrict__ cb = col + ebase;
        auto load = [&](int32_t wbase, Row& R) {
            R.i = wbase + sub;
            R.len = 0;
            if (R.i < c1) {
                const int32_t e0 = rp[R.i - c0];  // shared-memory row offsets: no dependent global load
                R.len = rp[R.i - c0 + 1] - e0;
#pragma unroll
                for (int j = 0; j < ROWCH; ++j) {
                    const int k = sl + j * VL;
                    const bool in = k < R.len;
                    R.v[j] = in ? vb[e0 + k] : (T)0;
                    R.c[j] = in ? cb[e0 + k] : (uint16_t)0;
                }
            }
        };
        auto process = [&](const Row& A) {
            T part = (T)0;
#pragma unroll
            for (int j = 0; j < ROWCH; ++j)
                if (sl + j * VL < A.len) part += A.v[j] * xs[A.c[j]];
            // lane partials and the butterfly in the storage precision, the row sum in fp64
            const double s = (double)group_sum_t<VL>(part);
            if (A.i < c1 && sl == 0) {
                const int32_t i = A.i;
                const double bi = NB ? (double)ob[i - c0] : 0.0, di = ND ? (double)od[i - c0] : 0.0,
                             ai = NA ? (double)oa[i - c0] : 0.0;
                if (MODE == PASS_JACOBI || MODE == PASS_JACOBI_DOT) {
                    T yi = (T)relax((double)xs[i - lo], i, omega, alpha, xprev, di, bi, s);
                    y[i] = yi;
                    if (MODE == PASS_JACOBI_DOT) { acc1 += ai * (double)yi; acc2 += ai * ai; }
                } else if (MODE == PASS_RESID_P) {
                    y[i] = (T)(ai * (bi - s));
                } else if (MODE == PASS_SPMV_DOT) {
                    T yi = (T)s;
                    y[i] = yi;
                    acc1 += (double)xs[i - lo] * (double)yi;
                } else if (MODE == PASS_POWER) {
                    T yi = (T)(di * s);
                    y[i] = yi;
                    acc1 += (double)yi * (double)yi;
                }
            }
        };
        // three rows in flight per group, rotated in place (no register copies)
        Row A, B, D;
        int32_t wb = c0 + warp * SPW;  // warp-uniform base row of this warp's current step
        load(wb, A);
        load(wb + NSLOT, B);
        load(wb + 2 * NSLOT, D);
        // single-exit loop with a warp-uniform trip count (rows past c1 are empty), so the butterfly
        // needs no divergence handling
        const int nsteps = wb < c1 ? (c1 - wb + NSLOT - 1) / NSLOT : 0;
        for (int t = 0; t < nsteps; t += 3) {
            process(A);
            load(wb + 3 * NSLOT, A);
            process(B);
            load(wb + 4 * NSLOT, B);
            process(D);
            load(wb + 5 * NSLOT, D);
            wb += 3 * NSLOT;
        }
    }
    if (MODE == PASS_JACOBI_DOT || MODE == PASS_SPMV_DOT || MODE == PASS_POWER) {
        __shared__ double sh[32];
        double t1 = block_sum<BB>(acc1, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t1;
        if (MODE == PASS_JACOBI_DOT) {
            double t2 = block_sum<BB>(acc2, sh);
            if (threadIdx.x == 0) parts2[blockIdx.x] = t2;
        }
    }
}

template <class T, int MODE, int VL>
void launch_rows(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                 double* parts2, cudaStream_t s) {
    const size_t smem = ((((size_t)A.band_rows + 1) * sizeof(int32_t) + 15) & ~(size_t)15) +
                        ((size_t)3 * A.band_rows + A.band_win) * sizeof(T);
    ensure_dyn_smem((const void*)k_rows<T, VL, MODE>, smem);
    k_rows<T, VL, MODE><<<A.band_grid, BB, smem, s>>>(A.row0, A.row0 + A.n, A.band_rows, A.win_lo, A.win_len, A.rowptr, A.col16,
                                                     A.val, A.dinv, x, b, y, aux, omega, alpha, xprev, parts, parts2);
    MG_LAUNCH_CHECK();
}

template <class T, int MODE>
void launch_rows_mode(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                      double* parts2, cudaStream_t s) {
    switch (A.row_vl) {
        case 4: launch_rows<T, MODE, 4>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 8: launch_rows<T, MODE, 8>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 16: launch_rows<T, MODE, 16>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        default: launch_rows<T, MODE, 32>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
    }
}

template <class T, int MODE, int VLR>
void launch_band(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                 double* parts2, cudaStream_t s) {
    const size_t smem = ((size_t)A.prod_cap + 8 + A.band_win) * sizeof(T);
    ensure_dyn_smem((const void*)k_band<T, VLR, MODE>, smem);
    k_band<T, VLR, MODE><<<A.band_grid, BB, smem, s>>>(A.row0, A.row0 + A.n, A.band_rows, A.win_lo, A.win_len, A.prod_cap, A.rowptr,
                                                      A.col, A.val, A.dinv, x, b, y, aux, omega, alpha, xprev, parts, parts2);
    MG_LAUNCH_CHECK();
}

template <class T, int MODE>
void launch_band_mode(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                      double* parts2, cudaStream_t s) {
    switch (A.vlr) {
        case 1: launch_band<T, MODE, 1>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 2: launch_band<T, MODE, 2>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 4: launch_band<T, MODE, 4>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 8: launch_band<T, MODE, 8>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 16: launch_band<T, MODE, 16>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        default: launch_band<T, MODE, 32>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
    }
}

// per band tile: the column window [min col, max col] of its rows (diagonal-last CSR)
__global__ void k_band_windows(int32_t row0, int32_t n, int32_t C, const int64_t* __restrict__ rowptr,
                               const int32_t* __restrict__ col, int32_t* __restrict__ lo, int32_t* __restrict__ hi) {
    int32_t li = blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= n) return;
    const int32_t i = row0 + li;
    const int64_t a = rowptr[i], z = rowptr[i + 1];
    int32_t mn = i, mx = i;
    if (z - a > 1) {
        mn = min(mn, col[a]);
        mx = max(mx, col[z - 2]);
    }
    atomicMin(&lo[li / C], mn);
    atomicMax(&hi[li / C], mx);
}
__global__ void k_band_len(int32_t nb, int32_t* __restrict__ lo, const int32_t* __restrict__ hi, int32_t* len,
                           int32_t* maxlen) {
    int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nb) return;
    len[t] = hi[t] - lo[t] + 1;
    atomicMax(maxlen, len[t]);
}

template <class T, int MODE, int VLR>
void launch_tile(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                 double* parts2, cudaStream_t s) {
    const size_t smem = (size_t)A.tile_nnz * sizeof(double);
    ensure_dyn_smem((const void*)k_tile<T, VLR, MODE>, smem);
    k_tile<T, VLR, MODE><<<A.grid, PB, smem, s>>>(A.row0, A.row0 + A.n, A.rowptr, A.col, A.val, A.dinv, x, b, y, aux, omega, alpha, xprev, parts, parts2);
    MG_LAUNCH_CHECK();
}

template <class T, int MODE>
void launch_tile_mode(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                      double* parts2, cudaStream_t s) {
    switch (A.vlr) {
        case 1: launch_tile<T, MODE, 1>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 2: launch_tile<T, MODE, 2>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 4: launch_tile<T, MODE, 4>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 8: launch_tile<T, MODE, 8>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case 16: launch_tile<T, MODE, 16>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        default: launch_tile<T, MODE, 32>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
    }
}

__global__ void k_max_tile(int32_t n, int R, const int64_t* __restrict__ rowptr, int32_t* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t r0 = t * R;
    if (r0 >= n) return;
    int64_t r1 = r0 + R < n ? r0 + R : n;
    atomicMax(out, (int32_t)(rowptr[r1] - rowptr[r0]));
}

template <class T, int MODE>
void launch_pass_mode(const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double alpha, const T* xprev, double* parts,
                      double* parts2, cudaStream_t s) {
#define MG_P(VL) k_pass<T, VL, MODE><<<A.grid, PB, 0, s>>>(A.row0, A.row0 + A.n, A.rowptr, A.col, A.val, A.dinv, x, b, y, aux, omega, alpha, xprev, parts, parts2)
    switch (A.vl) {
        case 2: MG_P(2); break;
        case 4: MG_P(4); break;
        case 8: MG_P(8); break;
        case 16: MG_P(16); break;
        default: MG_P(32); break;
    }
#undef MG_P
    MG_LAUNCH_CHECK();
}

// Streaming vector kernels: one 16-byte chunk (W elements) per thread, every load of the chunk issued before
// any arithmetic; V = false (an operand not 16-byte aligned, e.g. a rank's row offset) falls back to W = 1.
template <class T, bool V>
struct Chunk16 {
    static constexpr int W = V ? 16 / (int)sizeof(T) : 1;
    using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    // element range of chunk c: [c W, min(n, c W + W))
    __device__ static __forceinline__ bool full(int64_t c, int64_t n) { return (c + 1) * W <= n; }
    __device__ static __forceinline__ void ld(const T* __restrict__ a, int64_t c, int64_t n, T (&o)[W]) {
        if (V && full(c, n)) {
            const VT v = *reinterpret_cast<const VT*>(a + c * W);
            memcpy(o, &v, 16);
        } else {
#pragma unroll
            for (int w = 0; w < W; ++w) o[w] = c * W + w < n ? a[c * W + w] : (T)0;
        }
    }
    __device__ static __forceinline__ void st(T* __restrict__ a, int64_t c, int64_t n, const T (&o)[W]) {
        if (V && full(c, n)) {
            VT v;
            memcpy(&v, o, 16);
            *reinterpret_cast<VT*>(a + c * W) = v;
        } else {
#pragma unroll
            for (int w = 0; w < W; ++w)
                if (c * W + w < n) a[c * W + w] = o[w];
        }
    }
};
inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
template <class T, bool V>
inline int chunk_grid(int64_t n, int cpt = 1) {
    const int64_t items = (n + Chunk16<T, V>::W - 1) / Chunk16<T, V>::W;
    return (int)std::max<int64_t>(1, (items + (int64_t)PB * cpt - 1) / ((int64_t)PB * cpt));
}
// chunks per thread of the PCG update kernels (MGPBD_VEC_CPT: 1 or 4)
inline int vec_cpt() {
    const char* e = std::getenv("MGPBD_VEC_CPT");  // read per call (launch/capture time): tests toggle it
    const int c = e ? std::atoi(e) : 4;
    return c == 1 || c == 2 || c == 8 ? c : 4;
}

// The PCG vector kernels that precede a level-0 pass (Jacobi-0, prolongation, p update, x / r update) release
// the pass's PDL-launched vertex gather at their start: its persistent CTAs (one per SM, the whole register
// file) become resident as this grid's CTAs leave each SM, run their static prologue and wait in
// griddepcontrol.wait for this grid's completion (MGPBD_VEC_TRIGGER=0: released at exit).
#ifndef MGPBD_VEC_TRIGGER
#define MGPBD_VEC_TRIGGER 1
#endif
#define MG_VEC_TRIGGER()                                                                 \
    do {                                                                                 \
        if (MGPBD_VEC_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)

template <class T, bool V>
__global__ void k_jacobi0(int32_t n, const T* __restrict__ dinv, const T* __restrict__ b, double omega, T* __restrict__ y) {
    MG_VEC_TRIGGER();
    using C = Chunk16<T, V>;
    const int64_t c = blockIdx.x * (int64_t)PB + threadIdx.x;
    if (c * C::W >= n) return;
    T d[C::W], bb[C::W], o[C::W];
    C::ld(dinv, c, n, d);
    C::ld(b, c, n, bb);
#pragma unroll
    for (int w = 0; w < C::W; ++w) o[w] = (T)(omega * (double)d[w] * (double)bb[w]);
    C::st(y, c, n, o);
}

// bc[a] = sum_{i in a, ascending} t[i]: 8 lanes per aggregate, each lane's members in chunks of 4 with
// all list loads issued before the t gathers; lane partials + fixed-order butterfly (deterministic)
template <class T, int G, int UN = 4>
__global__ void k_restrict(int32_t nc, const int64_t* __restrict__ mptr, const int32_t* __restrict__ mlist,
                           const T* __restrict__ t, T* __restrict__ bc) {
    constexpr int PER = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * PER; base < nc; base += nw * PER) {  // warp-uniform trip count
        const int64_t a = base + sub;
        double s = 0.0;
        if (a < nc) {
            const int64_t m0 = mptr[a], m1 = mptr[a + 1];
            for (int64_t eb = m0 + sl; eb < m1; eb += G * UN) {
                int32_t mi[UN];
#pragma unroll
                for (int q = 0; q < UN; ++q) mi[q] = eb + q * G < m1 ? mlist[eb + q * G] : -1;
#pragma unroll
                for (int q = 0; q < UN; ++q) s += mi[q] >= 0 ? (double)t[mi[q]] : 0.0;
            }
        }
        s = group_sum<G>(s);
        if (a < nc && sl == 0) bc[a] = (T)s;
    }
}

template <class T, bool V>
__global__ void k_prolong(int32_t n, const int32_t* __restrict__ agg, const T* __restrict__ P, const T* __restrict__ e,
                          T* __restrict__ x) {
    MG_VEC_TRIGGER();
    using C = Chunk16<T, V>;
    constexpr int W = C::W;
    const int64_t c = blockIdx.x * (int64_t)PB + threadIdx.x;
    if (c * W >= n) return;
    T xv[W], pv[W], ev[W];
    int32_t ag[W];
    C::ld(x, c, n, xv);
    C::ld(P, c, n, pv);
    if (V && C::full(c, n)) {  // W 32-bit aggregate ids: 16 (fp32) or 8 bytes (fp64)
        if constexpr (W == 4) {
            const int4 a4 = *reinterpret_cast<const int4*>(agg + c * W);
            memcpy(ag, &a4, 16);
        } else if constexpr (W == 2) {
            const int2 a2 = *reinterpret_cast<const int2*>(agg + c * W);
            memcpy(ag, &a2, 8);
        } else {
            ag[0] = agg[c];
        }
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) ag[w] = c * W + w < n ? agg[c * W + w] : 0;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) ev[w] = e[ag[w]];
#pragma unroll
    for (int w = 0; w < W; ++w) xv[w] = (T)((double)xv[w] + (double)pv[w] * (double)ev[w]);
    C::st(x, c, n, xv);
}

// Convergence exit of MGPCG (pcg_tol > 0): true if the solve is frozen at iteration k, i.e. it was
// already converged or ||r_k||^2 = rr <= tol^2 ||b||^2 (||b||^2 = rr at k = 0).  The caller publishes
// ||b||^2 and the flag (one thread) and every thread takes the same decision.
__device__ __forceinline__ bool pcg_converged(const double* scal, int k, double rr) {
    if (scal[SC_DONE] != 0.0) return true;
    const double tol = scal[SC_TOL];
    if (!(tol > 0.0)) return false;
    const double b2 = k == 0 ? rr : scal[SC_B2];
    return rr <= tol * tol * b2;
}

template <class T>
__global__ void k_pcg_p(int32_t n, const T* __restrict__ z, T* __restrict__ p, const double* __restrict__ scal, int k) {
    if (scal[SC_DONE] != 0.0) return;  // converged (pcg_tol): the remaining iterations change nothing
    double beta = 0.0;
    if (k > 0) {
        double prev = scal[2 * (k - 1)];
        beta = prev != 0.0 ? scal[2 * k] / prev : 0.0;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (T)((double)z[i] + beta * (double)p[i]);
}

template <class T>
__global__ void k_pcg_xr(int32_t n, const T* __restrict__ p, const T* __restrict__ q, T* __restrict__ x,
                         T* __restrict__ r, const double* __restrict__ scal, int k) {
    if (scal[SC_DONE] != 0.0) return;
    double pq = scal[2 * k + 1];
    double alpha = pq != 0.0 ? scal[2 * k] / pq : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = (T)((double)x[i] + alpha * (double)p[i]);
        r[i] = (T)((double)r[i] - alpha * (double)q[i]);
    }
}

// Finalisation of <r,z> (and <r,r>) fused into the p update: every CTA reduces the partials in the same
// fixed order (identical value everywhere), CTA 0 publishes the scalar and raises the flags of
// k_fin_rz; saves one launch per PCG iteration.
template <class T, bool V, int CPT>
__global__ void k_pcg_p_fin(int32_t n, const T* __restrict__ z, T* __restrict__ p, double* __restrict__ scal, int k,
                            const double* __restrict__ prz, const double* __restrict__ prr, int np, int* flags,
                            int tag, const double* __restrict__ fin) {
    MG_VEC_TRIGGER();
    using CK = Chunk16<T, V>;
    constexpr int W = CK::W;
    // CPT chunks per thread (chunk c of the block strided by PB: coalesced), all loaded before the partial sums,
    // which every CTA reduces redundantly (fewer CTAs: less of that L2 traffic)
    T zv[CPT][W], pv[CPT][W];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int64_t ci = ((int64_t)blockIdx.x * CPT + c) * PB + threadIdx.x;
        if (ci * W < n) { CK::ld(z, ci, n, zv[c]); CK::ld(p, ci, n, pv[c]); }
    }
    __shared__ double sh[32];
    __shared__ double rz_s;
    double a = 0.0, c = 0.0;
    if (fin) {  // already summed by the producing row kernel's last CTA
        a = fin[0];
        c = fin[1];
    } else {
        for (int i = threadIdx.x; i < np; i += PB) { a += prz[i]; c += prr[i]; }
        a = block_sum<PB>(a, sh);
        c = block_sum<PB>(c, sh);
    }
    __shared__ int conv;
    if (threadIdx.x == 0) conv = pcg_converged(scal, k, c) ? 1 : 0;
    __syncthreads();
    if (conv) {  // converged: publish the flag, no event checks, no update
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (k == 0) scal[SC_B2] = c;
            scal[SC_DONE] = 1.0;
        }
        return;
    }
    if (threadIdx.x == 0) {
        rz_s = a;
        if (blockIdx.x == 0) {
            if (k == 0) scal[SC_B2] = c;
            scal[2 * k] = a;
            if (!isfinite(a) || !isfinite(c)) {
                if (atomicCAS(&flags[1], 0, 1) == 0) flags[3] = flags[7] * 4096 + tag;
            } else if (a < 0.0 || (a == 0.0 && c > 0.0)) {
                if (atomicCAS(&flags[0], 0, 1) == 0) flags[2] = flags[7] * 4096 + tag;
                atomicAdd(&flags[4], 1);
            }
        }
    }
    __syncthreads();
    double beta = 0.0;
    if (k > 0) {
        const double prev = scal[2 * (k - 1)];
        beta = prev != 0.0 ? rz_s / prev : 0.0;
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int64_t ci = ((int64_t)blockIdx.x * CPT + c) * PB + threadIdx.x;
        if (ci * W >= n) break;
#pragma unroll
        for (int w = 0; w < W; ++w) pv[c][w] = (T)((double)zv[c][w] + beta * (double)pv[c][w]);
        CK::st(p, ci, n, pv[c]);
    }
}

// <p,q> finalisation fused into the x / r update (see k_pcg_p_fin)
template <class T, bool V, int CPT>
__global__ void k_pcg_xr_fin(int32_t n, const T* __restrict__ p, const T* __restrict__ q, T* __restrict__ x,
                             T* __restrict__ r, double* __restrict__ scal, int k, const double* __restrict__ ppq,
                             int np, int* flags, int tag, const T* __restrict__ dinv, double om0, T* __restrict__ x1,
                             const double* __restrict__ fin) {
    MG_VEC_TRIGGER();
    if (scal[SC_DONE] != 0.0) return;
    using CK = Chunk16<T, V>;
    constexpr int W = CK::W;
    T xv[CPT][W], pv[CPT][W], rv[CPT][W], qv[CPT][W], dv[CPT][W];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {  // issued before the partial sums
        const int64_t ci = ((int64_t)blockIdx.x * CPT + c) * PB + threadIdx.x;
        if (ci * W < n) {
            CK::ld(x, ci, n, xv[c]); CK::ld(p, ci, n, pv[c]); CK::ld(r, ci, n, rv[c]); CK::ld(q, ci, n, qv[c]);
            if (x1) CK::ld(dinv, ci, n, dv[c]);
        }
    }
    __shared__ double sh[32];
    __shared__ double pq_s;
    double a = 0.0;
    if (fin) {
        a = fin[2];
    } else {
        for (int i = threadIdx.x; i < np; i += PB) a += ppq[i];
        a = block_sum<PB>(a, sh);
    }
    if (threadIdx.x == 0) {
        pq_s = a;
        if (blockIdx.x == 0) {
            scal[2 * k + 1] = a;
            if (!isfinite(a))
                if (atomicCAS(&flags[1], 0, 1) == 0) flags[3] = flags[7] * 4096 + tag;
        }
    }
    __syncthreads();
    const double alpha = pq_s != 0.0 ? scal[2 * k] / pq_s : 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int64_t ci = ((int64_t)blockIdx.x * CPT + c) * PB + threadIdx.x;
        if (ci * W >= n) break;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            xv[c][w] = (T)((double)xv[c][w] + alpha * (double)pv[c][w]);
            rv[c][w] = (T)((double)rv[c][w] - alpha * (double)qv[c][w]);
        }
        CK::st(x, ci, n, xv[c]);
        CK::st(r, ci, n, rv[c]);
        if (x1) {  // the next V-cycle's step 0 (k_jacobi0's expression on the new residual)
#pragma unroll
            for (int w = 0; w < W; ++w) dv[c][w] = (T)(om0 * (double)dv[c][w] * (double)rv[c][w]);
            CK::st(x1, ci, n, dv[c]);
        }
    }
}

// One colour of a multicolour Gauss-Seidel sweep (reading c22): for the rows of colour c
// (mutually independent), x_i = (b_i - sum_{j != i} A_ij x_j) / A_ii in place; warp per row, diagonal
// last in every row; products in T, row sum in fp64.
template <class T>
__global__ void k_gs_colour_smooth(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                   const T* __restrict__ val, const int64_t* __restrict__ gs_ptr,
                                   const int32_t* __restrict__ gs_list, int c, const T* __restrict__ b,
                                   T* __restrict__ x) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t r0 = gs_ptr[c], r1 = gs_ptr[c + 1];
    for (int64_t t = r0 + gw; t < r1; t += nw) {
        const int32_t i = gs_list[t];
        const int64_t a = rowptr[i], e = rowptr[i + 1] - 1;
        T part = (T)0;
        for (int64_t k = a + lane; k < e; k += 32) part += val[k] * x[col[k]];
        const double sum = group_sum<32>((double)part);
        if (lane == 0) x[i] = (T)(((double)b[i] - sum) / (double)val[e]);
    }
}

template <class T>
__global__ void k_dot(int32_t n, const T* __restrict__ a, const T* __restrict__ b, double* __restrict__ parts) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v += (double)a[i] * (double)b[i];
    v = block_sum<PB>(v, sh);
    if (threadIdx.x == 0) parts[blockIdx.x] = v;
}

template <class T>
__global__ void k_scale(int32_t n, const T* __restrict__ w, T* __restrict__ v, const double* __restrict__ ss) {
    double lam = sqrt(*ss);
    double inv = lam > 0.0 ? 1.0 / lam : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (T)((double)w[i] * inv);
}

__global__ void k_fin_rz(const double* __restrict__ prz, const double* __restrict__ prr, int np, double* scal, int k,
                         int* flags, int tag) {
    __shared__ double sh[32];
    double a = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < np; i += 1024) { a += prz[i]; c += prr[i]; }
    a = block_sum<1024>(a, sh);
    c = block_sum<1024>(c, sh);
    if (threadIdx.x == 0) {
        const bool conv = pcg_converged(scal, k, c);
        if (k == 0) scal[SC_B2] = c;
        if (conv) { scal[SC_DONE] = 1.0; return; }
        scal[2 * k] = a;
        if (!isfinite(a) || !isfinite(c)) {
            if (atomicCAS(&flags[1], 0, 1) == 0) flags[3] = flags[7] * 4096 + tag;
        } else if (a < 0.0 || (a == 0.0 && c > 0.0)) {
            if (atomicCAS(&flags[0], 0, 1) == 0) flags[2] = flags[7] * 4096 + tag;
            atomicAdd(&flags[4], 1);
        }
    }
}
__global__ void k_fin_pq(const double* __restrict__ p, int np, double* scal, int k, int* flags, int tag) {
    __shared__ double sh[32];
    double a = 0.0;
    for (int i = threadIdx.x; i < np; i += 1024) a += p[i];
    a = block_sum<1024>(a, sh);
    if (threadIdx.x == 0) {
        scal[2 * k + 1] = a;
        if (!isfinite(a)) {
            if (atomicCAS(&flags[1], 0, 1) == 0) flags[3] = flags[7] * 4096 + tag;
        }
    }
}

// Gauss-Jordan in-place inversion of the dense SPD coarsest matrix, one CTA.
template <class T>
__global__ void __launch_bounds__(1024) k_coarse_inv(int32_t n, const int64_t* __restrict__ rowptr,
                                                     const int32_t* __restrict__ col, const T* __restrict__ val,
                                                     double* __restrict__ gwork, double* __restrict__ Ainv,
                                                     int* flags, int use_smem) {
    extern __shared__ double smem[];
    double* W = use_smem ? smem : gwork;
    const int64_t nn = (int64_t)n * n;
    for (int64_t k = threadIdx.x; k < nn; k += blockDim.x) W[k] = 0.0;
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x)
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) W[(int64_t)i * n + col[e]] = (double)val[e];
    __syncthreads();
    __shared__ double piv_s;
    for (int32_t k = 0; k < n; ++k) {
        if (threadIdx.x == 0) {
            double p = W[(int64_t)k * n + k];
            if (!(p > 0.0)) {
                flags[5] = 1;
                p = (p == 0.0 || !isfinite(p)) ? 1.0 : p;
            }
            piv_s = p;
        }
        __syncthreads();
        const double ip = 1.0 / piv_s;
        {   // warp per row, lanes over columns (no 64-bit index division: it dominated this loop)
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
            const double* __restrict__ Wk = W + (int64_t)k * n;
            for (int32_t i = warp; i < n; i += nw) {
                if (i == k) continue;
                double* Wi = W + (int64_t)i * n;
                const double wik = Wi[k];
                for (int32_t j = lane; j < n; j += 32)
                    if (j != k) Wi[j] -= wik * Wk[j] * ip;
            }
        }
        __syncthreads();
        for (int32_t t = threadIdx.x; t < n; t += blockDim.x) {
            if (t != k) {
                W[(int64_t)k * n + t] *= ip;
                W[(int64_t)t * n + k] = -W[(int64_t)t * n + k] * ip;
            }
        }
        if (threadIdx.x == 0) W[(int64_t)k * n + k] = ip;
        __syncthreads();
    }
    for (int64_t k = threadIdx.x; k < nn; k += blockDim.x) Ainv[k] = W[k];
}

// ---- blocked Gauss-Jordan (block size GJB) for coarsest levels too large for one CTA's smem.
// Step k (block K = [k0, k0+bs)): P = W_KK^-1; R = P W_K,: ; C = W_:,K (old);
// W_ij -= C_i R_j (i,j not in K); W_Kj = R_j; W_iK = -C_i P; W_KK = P.  SPD => no pivoting.
constexpr int GJB = 32;

template <class T>
__global__ void k_dense_load(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                             const T* __restrict__ val, double* __restrict__ W) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < n; i += nw) {
        for (int32_t j = lane; j < n; j += 32) W[i * n + j] = 0.0;
        __syncwarp();
        for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) W[i * n + col[e]] = (double)val[e];
    }
}

__global__ void __launch_bounds__(1024) k_gj_diag(int32_t n, const double* __restrict__ W, int32_t k0, int32_t bs,
                                                  double* __restrict__ P, int* flags) {
    __shared__ double S[GJB * GJB];
    __shared__ double piv;
    const int t = threadIdx.x;
    if (t < bs * bs) S[t] = W[(int64_t)(k0 + t / bs) * n + k0 + t % bs];
    __syncthreads();
    for (int k = 0; k < bs; ++k) {
        if (t == 0) {
            double p = S[k * bs + k];
            if (!(p > 0.0)) { flags[5] = 1; p = (p == 0.0 || !isfinite(p)) ? 1.0 : p; }
            piv = p;
        }
        __syncthreads();
        const double ip = 1.0 / piv;
        double upd = 0.0;
        const int i = t / bs, j = t % bs;
        if (t < bs * bs && i != k && j != k) upd = S[i * bs + j] - S[i * bs + k] * S[k * bs + j] * ip;
        __syncthreads();
        if (t < bs * bs) {
            if (i != k && j != k) S[t] = upd;
            else if (i == k && j != k) S[t] = S[t] * ip;
            else if (i != k && j == k) S[t] = -S[t] * ip;
            else S[t] = ip;
        }
        __syncthreads();
    }
    if (t < bs * bs) P[t] = S[t];
}

// R[t][j] = sum_s P[t][s] W[k0+s][j] (j not in K);  C[i][t] = W[i][k0+t] (i not in K)
__global__ void k_gj_panel(int32_t n, const double* __restrict__ W, int32_t k0, int32_t bs, const double* __restrict__ P,
                           double* __restrict__ C, double* __restrict__ R) {
    const int64_t tot = (int64_t)n * bs;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < 2 * tot; q += (int64_t)gridDim.x * blockDim.x) {
        if (q < tot) {
            const int32_t t = (int32_t)(q / n), j = (int32_t)(q % n);
            if (j >= k0 && j < k0 + bs) continue;
            double s = 0.0;
            for (int u = 0; u < bs; ++u) s += P[t * bs + u] * W[(int64_t)(k0 + u) * n + j];
            R[(int64_t)t * n + j] = s;
        } else {
            const int64_t q2 = q - tot;
            const int32_t i = (int32_t)(q2 / bs), t = (int32_t)(q2 % bs);
            if (i >= k0 && i < k0 + bs) continue;
            C[(int64_t)i * bs + t] = W[(int64_t)i * n + k0 + t];
        }
    }
}

// 32x32 output tile per CTA (32x8 threads, 4 outputs each)
__global__ void __launch_bounds__(256) k_gj_update(int32_t n, double* __restrict__ W, int32_t k0, int32_t bs,
                                                   const double* __restrict__ P, const double* __restrict__ C,
                                                   const double* __restrict__ R) {
    __shared__ double Cs[32][GJB + 1];
    __shared__ double Rs[GJB][32 + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int32_t i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    for (int r = ty; r < 32; r += 8) {
        const int32_t i = i0 + r;
        Cs[r][tx] = (i < n && tx < bs && !(i >= k0 && i < k0 + bs)) ? C[(int64_t)i * bs + tx] : 0.0;
        const int32_t j = j0 + tx;
        if (r < bs) Rs[r][tx] = (j < n && !(j >= k0 && j < k0 + bs)) ? R[(int64_t)r * n + j] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int32_t i = i0 + r, j = j0 + tx;
        if (i >= n || j >= n) continue;
        const bool iK = i >= k0 && i < k0 + bs, jK = j >= k0 && j < k0 + bs;
        double* w = &W[(int64_t)i * n + j];
        if (!iK && !jK) {
            double s = 0.0;
            for (int t = 0; t < bs; ++t) s += Cs[r][t] * Rs[t][tx];
            *w -= s;
        } else if (iK && !jK) {
            *w = R[(int64_t)(i - k0) * n + j];
        } else if (!iK && jK) {
            double s = 0.0;
            for (int t = 0; t < bs; ++t) s += Cs[r][t] * P[t * bs + (j - k0)];
            *w = -s;
        } else {
            *w = P[(i - k0) * bs + (j - k0)];
        }
    }
}

// The same panel update for large n (the k > 1 hierarchies' coarsest levels of 2-8K rows, where the cooperative
// kernel recomputes R = P K in every 32 x 32 tile and streams its operands at two shared loads per FMA): 64 x 64
// output tile per CTA of 512 threads, thread (tx, ty) of 32 x 16 owns rows ty + 16a (a < 4) and columns tx + 32b
// (b < 2), so each k step is 6 shared loads (broadcast / consecutive) for 8 FMAs; the thread's old W values are
// loaded before the staging.  Columns j in K take P in place of R, so the same accumulation gives C P there.  Same
// outputs as k_gj_update (sums over t in the same order).  n = 7656 (k = 6 bench hierarchy), per inverse: 118 ms
// with 256 threads x 16 outputs, 110 with the early W loads, 94 with 512 threads at 2 CTAs per SM (1 CTA per SM
// at 108 registers: 148; 3 CTAs at 40 registers: 100).
#ifndef MGPBD_GJ_PREFETCH
#define MGPBD_GJ_PREFETCH 1
#endif
#ifndef MGPBD_GJU_T
#define MGPBD_GJU_T 512
#endif
#ifndef MGPBD_GJU_MINB
#define MGPBD_GJU_MINB 2
#endif
constexpr int GJU_T = MGPBD_GJU_T;           // threads per CTA: 256 (4 x 4 outputs each) or 512 (4 x 2)
constexpr int GJU_CX = GJU_T == 512 ? 32 : 16;  // thread columns
constexpr int GJU_NB = 64 / GJU_CX;             // columns per thread
__global__ void __launch_bounds__(GJU_T, MGPBD_GJU_MINB) k_gj_update64(int32_t n, double* __restrict__ W, int32_t k0, int32_t bs,
                                                       const double* __restrict__ P, const double* __restrict__ C,
                                                       const double* __restrict__ R) {
    __shared__ double Cs[64][GJB + 1];
    __shared__ double Rs[GJB][64 + 1];
    const int t = threadIdx.x, tx = t % GJU_CX, ty = t / GJU_CX;
    const int32_t i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
    // the old values this thread updates are loaded first: their HBM latency overlaps the staging + products
    double wold[4][GJU_NB];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < GJU_NB; ++b) {
            const int32_t i = i0 + ty + 16 * a, j = j0 + tx + GJU_CX * b;
            wold[a][b] = (MGPBD_GJ_PREFETCH && i < n && j < n) ? W[(int64_t)i * n + j] : 0.0;
        }
    for (int q = t; q < 64 * GJB; q += GJU_T) {
        const int r = q / GJB, u = q % GJB;  // C tile: row r, column u (coalesced over u)
        const int32_t i = i0 + r;
        Cs[r][u] = (i < n && u < bs && !(i >= k0 && i < k0 + bs)) ? C[(int64_t)i * bs + u] : 0.0;
        const int u2 = q / 64, c = q % 64;  // R tile: row u2, column c (coalesced over c)
        const int32_t j = j0 + c;
        double rv = 0.0;
        if (u2 < bs && j < n) rv = (j >= k0 && j < k0 + bs) ? P[u2 * bs + (j - k0)] : R[(int64_t)u2 * n + j];
        Rs[u2][c] = rv;
    }
    __syncthreads();
    double acc[4][GJU_NB] = {};
#pragma unroll 8
    for (int u = 0; u < GJB; ++u) {
        double cv[4], rv[GJU_NB];
#pragma unroll
        for (int a = 0; a < 4; ++a) cv[a] = Cs[ty + 16 * a][u];
#pragma unroll
        for (int b = 0; b < GJU_NB; ++b) rv[b] = Rs[u][tx + GJU_CX * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < GJU_NB; ++b) acc[a][b] += cv[a] * rv[b];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int32_t i = i0 + ty + 16 * a;
        if (i >= n) continue;
        const bool iK = i >= k0 && i < k0 + bs;
#pragma unroll
        for (int b = 0; b < GJU_NB; ++b) {
            const int32_t j = j0 + tx + GJU_CX * b;
            if (j >= n) continue;
            const bool jK = j >= k0 && j < k0 + bs;
            double* w = &W[(int64_t)i * n + j];
            if (!iK && !jK) *w = (MGPBD_GJ_PREFETCH ? wold[a][b] : *w) - acc[a][b];
            else if (iK && !jK) *w = R[(int64_t)(i - k0) * n + j];
            else if (!iK && jK) *w = -acc[a][b];
            else *w = P[(i - k0) * bs + (j - k0)];
        }
    }
}

// Blocked Gauss-Jordan inverse as ONE cooperative kernel (one grid barrier per 32-wide panel instead of
// three launches).  Ping-pong between two n x n buffers so no tile reads a value another CTA writes in
// the same panel.  Every CTA inverts the 32x32 pivot block itself (all 256 threads, 4 entries each,
// two shared buffers alternating so each elimination step needs one barrier), then updates its 32x32
// output tiles (thread (ty, lane) owns rows ty, ty+8, ty+16, ty+24 of column lane: 4 independent
// accumulators):
//   i,j outside K: W' = W - C R,  i in K: W' = R,  j in K: W' = -C P,  both: W' = P
// with P = (W_KK)^-1, C = W_{:,K}, R = P W_{K,:}.  (tools/micro/gj.cu: 268 -> 190 us at n = 357.)
constexpr int GJT = 256;
template <class T>
__global__ void __launch_bounds__(GJT) k_gj_coop(int32_t n, const int64_t* __restrict__ rowptr,
                                                 const int32_t* __restrict__ col, const T* __restrict__ val,
                                                 double* __restrict__ W0, double* __restrict__ W1, int* flags) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double Ps[32][33];
    __shared__ double Qs[32][33];
    __shared__ double Ks[32][33];  // W_old[K rows][J cols]
    __shared__ double Cs[32][33];  // W_old[I rows][K cols]
    __shared__ double Rs[32][33];
    const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int npan = (n + 31) / 32;
    double* cur = (npan % 2 == 0) ? W0 : W1;  // the buffer that holds the inverse after npan swaps is W0
    double* nxt = (npan % 2 == 0) ? W1 : W0;
    {
        const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
        for (int64_t i = gw; i < n; i += nw) {
            for (int32_t j = lane; j < n; j += 32) cur[i * n + j] = 0.0;
            __syncwarp();
            for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) cur[i * n + col[e]] = (double)val[e];
        }
    }
    grid.sync();
    for (int pnl = 0; pnl < npan; ++pnl) {
        const int32_t k0 = pnl * 32, bs = min(32, n - k0);
        // P = inverse of the pivot block (identity-padded to 32 x 32); step k reads one buffer, writes the other
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = ty + 8 * u;
            Ps[i][lane] = (i < bs && lane < bs) ? cur[(int64_t)(k0 + i) * n + k0 + lane] : (i == lane ? 1.0 : 0.0);
        }
        __syncthreads();
#pragma unroll 2
        for (int k = 0; k < 32; ++k) {
            double (*A_)[33] = (k & 1) ? Qs : Ps;
            double (*B_)[33] = (k & 1) ? Ps : Qs;
            double pv = A_[k][k];
            if (!(pv > 0.0)) {  // SPD: a non-positive pivot means the coarse matrix lost definiteness
                if (blockIdx.x == 0 && threadIdx.x == 0) flags[5] = 1;
                pv = (pv == 0.0 || !isfinite(pv)) ? 1.0 : pv;
            }
            const double ip = 1.0 / pv;
            const double akj = A_[k][lane] * ip;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = ty + 8 * u;
                const double aik = A_[i][k];
                double v;
                if (i == k) v = lane == k ? ip : akj;
                else v = lane == k ? -aik * ip : fma(-aik, akj, A_[i][lane]);
                B_[i][lane] = v;
            }
            __syncthreads();
        }  // 32 steps: the inverse is back in Ps
        const int nt = npan * npan;
        for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
            const int I = tile / npan, J = tile % npan;
            const int32_t i0 = I * 32, j0 = J * 32;
            const bool iK = I == pnl, jK = J == pnl;
            double old[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = ty + 8 * u;
                if (!jK) Ks[r][lane] = (r < bs && j0 + lane < n) ? cur[(int64_t)(k0 + r) * n + j0 + lane] : 0.0;
                if (!iK) Cs[r][lane] = (i0 + r < n && lane < bs) ? cur[(int64_t)(i0 + r) * n + k0 + lane] : 0.0;
                old[u] = (!iK && !jK && i0 + r < n && j0 + lane < n) ? cur[(int64_t)(i0 + r) * n + j0 + lane] : 0.0;
            }
            __syncthreads();
            if (!jK) {  // R = P K
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const double kv = Ks[t][lane];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = fma(Ps[ty + 8 * u][t], kv, acc[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) Rs[ty + 8 * u][lane] = acc[u];
            }
            __syncthreads();
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (!iK) {  // C R (j outside K) or C P (j in K)
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const double rv = jK ? Ps[t][lane] : Rs[t][lane];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = fma(Cs[ty + 8 * u][t], rv, acc[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = ty + 8 * u;
                const int32_t i = i0 + r, j = j0 + lane;
                if (i >= n || j >= n) continue;
                double v;
                if (iK && jK) v = Ps[r][lane];
                else if (iK) v = Rs[r][lane];
                else if (jK) v = -acc[u];
                else v = old[u] - acc[u];
                nxt[(int64_t)i * n + j] = v;
            }
            __syncthreads();
        }
        grid.sync();
        double* t = cur; cur = nxt; nxt = t;
    }
}

template <class T>
__global__ void k_coarse_gemv(int32_t n, const double* __restrict__ Ainv, const T* __restrict__ b, T* __restrict__ x) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = gw; i < n; i += nw) {
        double s = 0.0;
        for (int32_t j = lane; j < n; j += 32) s += Ainv[i * n + j] * (double)b[j];
        s = group_sum<32>(s);
        if (lane == 0) x[i] = (T)s;
    }
}

}  // namespace

void tile_config(int32_t n, int64_t nnz, const int64_t* rowptr, int& vlr, int& grid, int& tile_nnz, cudaStream_t s) {
    const double avg = n ? (double)nnz / n : 1.0;
    vlr = 1;
    while (vlr < 32 && vlr * 2 <= avg / 8.0) vlr *= 2;
    const int R = PB / vlr;
    const int64_t ntiles = ((int64_t)n + R - 1) / R;
    grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, 148 * 8));
    int32_t* d;
    MG_CK(cudaMallocAsync(&d, sizeof(int32_t), s));
    MG_CK(cudaMemsetAsync(d, 0, sizeof(int32_t), s));
    if (n) {
        k_max_tile<<<(int)((ntiles + 255) / 256), 256, 0, s>>>(n, R, rowptr, d);
        MG_LAUNCH_CHECK();
    }
    int32_t h = 0;
    MG_CK(cudaMemcpyAsync(&h, d, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MG_CK(cudaFreeAsync(d, s));
    MG_CK(cudaStreamSynchronize(s));
    tile_nnz = std::max(1, h);
    if ((size_t)tile_nnz * sizeof(double) > 200 * 1024) vlr = 0;  // fall back to the warp-per-row kernel
    // rows of >= 128 entries on average (vlr 16 / 32): the warp-per-row kernel k_pass, 32 lanes per row, streams
    // them far faster than the tile kernel, whose per-tile shared-memory products (25-50 KB) leave 4 CTAs per SM
    // with 3 serialised latencies per tile (k = 6 coarse levels of 200-600 entries per row: the 2-outer-iteration
    // frame 100.8 -> 61.1 ms, profiles/r2/experiments_log.txt); MGPBD_TILE_LONG_ROWS=1 keeps the tile kernel
    if (vlr >= 16 && !std::getenv("MGPBD_TILE_LONG_ROWS")) vlr = 0;
}

namespace {
__global__ void k_rowlen_max2(int32_t n, const int64_t* __restrict__ rowptr, int32_t* out) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMax(out, (int32_t)(rowptr[i + 1] - rowptr[i]));
}
}  // namespace

template <class T>
bool band_config(int32_t row0, int32_t n, const int64_t* rowptr, const int32_t* col, int vlr, DBuf<int32_t>& lo,
                 DBuf<int32_t>& len, int& C, int& grid, int& prod_cap, int& win, int& row_vl, DBuf<uint16_t>& col16,
                 cudaStream_t s) {
    C = 0;
    row_vl = 0;
    if (n < 4096 || vlr <= 0) return false;
    DBuf<int32_t> tmp, hi;
    tmp.resize(2);
    MG_CK(cudaMemsetAsync(tmp.p, 0, 2 * sizeof(int32_t), s));
    k_rowlen_max2<<<ceil_div(n, 256), 256, 0, s>>>(n, rowptr + row0, tmp.p);
    MG_LAUNCH_CHECK();
    int32_t maxrow = 0;
    MG_CK(cudaMemcpyAsync(&maxrow, tmp.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MG_CK(cudaStreamSynchronize(s));
    const int R = BB / vlr;
    prod_cap = R * maxrow;
    const size_t budget = 227 * 1024 - 2048;  // leave room for the kernel's static shared memory
    auto windows = [&](int32_t c) {
        const int32_t nb = (n + c - 1) / c;
        lo.resize(nb); hi.resize(nb); len.resize(nb);
        fill_i32(lo.p, INT32_MAX, nb, s);
        fill_i32(hi.p, -1, nb, s);
        k_band_windows<<<ceil_div(n, 256), 256, 0, s>>>(row0, n, c, rowptr, col, lo.p, hi.p);
        MG_LAUNCH_CHECK();
        MG_CK(cudaMemsetAsync(tmp.p + 1, 0, sizeof(int32_t), s));
        k_band_len<<<ceil_div(nb, 256), 256, 0, s>>>(nb, lo.p, hi.p, len.p, tmp.p + 1);
        MG_LAUNCH_CHECK();
        int32_t mw = 0;
        MG_CK(cudaMemcpyAsync(&mw, tmp.p + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        MG_CK(cudaStreamSynchronize(s));
        return mw;
    };
    // 1) barrier-free row kernel: VL lanes per row (rows of at most ROWCH*VL entries); shared memory
    //    holds the band tile's row offsets, its per-row operands and the x window.  Band tiles are
    //    sized so every CTA gets the same whole number of them (k per SM).
    {
        const double avg = (double)(read_scalar(rowptr + row0 + n, s) - read_scalar(rowptr + row0, s)) / n;
        int v = 4;
        while (v < 32 && v * 5 < avg) v *= 2;
        while (v < 32 && maxrow > ROWCH * v) v *= 2;
        if (maxrow <= ROWCH * v && !std::getenv("MGPBD_NO_ROWS")) {
            for (int k = 1; k <= 64; ++k) {
                const int32_t c = (int32_t)(((int64_t)n + 148 * k - 1) / (148 * k));
                const int32_t mw = windows(c);
                const size_t need = (((size_t)(c + 1) * 4 + 15) & ~(size_t)15) + ((size_t)3 * c + mw) * sizeof(T);
                if (mw <= 65536 && need <= budget) {
                    const int32_t nb = (n + c - 1) / c;
                    C = c; win = mw; grid = nb < 148 ? nb : 148; row_vl = v;
                    const int64_t nnz = read_scalar(rowptr + row0 + n, s);  // global positions up to the range end
                    col16.resize(nnz);
                    k_col16<<<(int)std::min<int64_t>(((int64_t)n * 32 + 255) / 256, 148 * 16), 256, 0, s>>>(
                        row0, n, c, rowptr, col, lo.p, col16.p);
                    MG_LAUNCH_CHECK();
                    MG_CK(cudaStreamSynchronize(s));
                    return true;
                }
            }
        }
    }
    // 2) band kernel with a shared product buffer
    if ((size_t)prod_cap * sizeof(T) >= budget || prod_cap + 6 > BAND_EPT * BB) return false;
    for (int32_t c = ((n + 147) / 148 + R - 1) / R * R; c >= R; c = (c / 2 + R - 1) / R * R) {
        const int32_t mw = windows(c);
        if ((size_t)(prod_cap + 8 + mw) * sizeof(T) <= budget) {
            const int32_t nb = (n + c - 1) / c;
            C = c; win = mw; grid = nb < 148 ? nb : 148;
            return true;
        }
        if (c == R) break;
    }
    return false;
}
template bool band_config<float>(int32_t, int32_t, const int64_t*, const int32_t*, int, DBuf<int32_t>&, DBuf<int32_t>&,
                                 int&, int&, int&, int&, int&, DBuf<uint16_t>&, cudaStream_t);
template bool band_config<double>(int32_t, int32_t, const int64_t*, const int32_t*, int, DBuf<int32_t>&,
                                  DBuf<int32_t>&, int&, int&, int&, int&, int&, DBuf<uint16_t>&, cudaStream_t);

namespace {
__global__ void k_commit_rz(const double* __restrict__ d2, double* scal, int k, int* flags, int tag) {
    const double a = d2[0], c = d2[1];
    const bool conv = pcg_converged(scal, k, c);
    if (k == 0) scal[SC_B2] = c;
    if (conv) { scal[SC_DONE] = 1.0; return; }
    scal[2 * k] = a;
    if (!isfinite(a) || !isfinite(c)) {
        if (atomicCAS(&flags[1], 0, 1) == 0) flags[3] = flags[7] * 4096 + tag;
    } else if (a < 0.0 || (a == 0.0 && c > 0.0)) {
        if (atomicCAS(&flags[0], 0, 1) == 0) flags[2] = flags[7] * 4096 + tag;
        atomicAdd(&flags[4], 1);
    }
}
__global__ void k_commit_pq(const double* __restrict__ d1, double* scal, int k, int* flags, int tag) {
    const double a = d1[0];
    scal[2 * k + 1] = a;
    if (!isfinite(a)) {
        if (atomicCAS(&flags[1], 0, 1) == 0) flags[3] = flags[7] * 4096 + tag;
    }
}
__global__ void k_range_window(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int32_t a,
                               int32_t b, int32_t* out) {
    int32_t i = a + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b) return;
    const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
    int32_t mn = i, mx = i;
    if (e1 - e0 > 1) { mn = min(mn, col[e0]); mx = max(mx, col[e1 - 2]); }
    atomicMin(&out[0], mn);
    atomicMax(&out[1], mx);
}
}  // namespace

__global__ void k_set_int(int* p, int v) { *p = v; }
void set_outer_index(int* flags, int ite, cudaStream_t s) {
    k_set_int<<<1, 1, 0, s>>>(flags + 7, ite);
    MG_LAUNCH_CHECK();
}
__global__ void k_pcg_begin(double* scal, double tol) {
    scal[SC_TOL] = tol;
    scal[SC_DONE] = 0.0;
}
void pcg_begin(double* scal, double tol, cudaStream_t s) {
    k_pcg_begin<<<1, 1, 0, s>>>(scal, tol);
    MG_LAUNCH_CHECK();
}
void pcg_commit_rz(const double* d2, double* scal, int k, int* flags, int tag, cudaStream_t s) {
    k_commit_rz<<<1, 1, 0, s>>>(d2, scal, k, flags, tag);
    MG_LAUNCH_CHECK();
}
void pcg_commit_pq(const double* d1, double* scal, int k, int* flags, int tag, cudaStream_t s) {
    k_commit_pq<<<1, 1, 0, s>>>(d1, scal, k, flags, tag);
    MG_LAUNCH_CHECK();
}
void row_range_window(const int64_t* rowptr, const int32_t* col, int32_t a, int32_t b, int32_t* lo, int32_t* hi,
                      cudaStream_t s) {
    DBuf<int32_t> d;
    d.resize(2);
    int32_t init[2] = {INT32_MAX, -1};
    h2d(d.p, init, 2, s);
    if (b > a) {
        k_range_window<<<ceil_div(b - a, 256), 256, 0, s>>>(rowptr, col, a, b, d.p);
        MG_LAUNCH_CHECK();
    }
    int32_t out[2];
    d2h(out, d.p, 2, s);
    MG_CK(cudaStreamSynchronize(s));
    *lo = out[0] == INT32_MAX ? a : out[0];
    *hi = out[1] < 0 ? a - 1 : out[1];
}

int pass_grid(int32_t n, int vl) {
    int rows_per_block = PB / vl;
    int64_t g = ((int64_t)n + rows_per_block - 1) / rows_per_block;
    if (g < 1) g = 1;
    return (int)(g < 148 * 8 ? g : 148 * 8);
}

template <class T>
void csr_pass(int mode, const Csr<T>& A, const T* x, const T* b, T* y, const T* aux, double omega, double* parts,
              double* parts2, cudaStream_t s, double alpha, const T* xprev) {
    if (A.n == 0) return;
    if (A.band_rows > 0 && A.row_vl > 0) {
        switch (mode) {
            case PASS_JACOBI: launch_rows_mode<T, PASS_JACOBI>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_JACOBI_DOT: launch_rows_mode<T, PASS_JACOBI_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_RESID_P: launch_rows_mode<T, PASS_RESID_P>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_SPMV_DOT: launch_rows_mode<T, PASS_SPMV_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_POWER: launch_rows_mode<T, PASS_POWER>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            default: throw Error(-1, "bad pass mode");
        }
        return;
    }
    if (A.band_rows > 0) {
        switch (mode) {
            case PASS_JACOBI: launch_band_mode<T, PASS_JACOBI>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_JACOBI_DOT: launch_band_mode<T, PASS_JACOBI_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_RESID_P: launch_band_mode<T, PASS_RESID_P>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_SPMV_DOT: launch_band_mode<T, PASS_SPMV_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_POWER: launch_band_mode<T, PASS_POWER>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            default: throw Error(-1, "bad pass mode");
        }
        return;
    }
    if (A.vlr > 0) {
        switch (mode) {
            case PASS_JACOBI: launch_tile_mode<T, PASS_JACOBI>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_JACOBI_DOT: launch_tile_mode<T, PASS_JACOBI_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_RESID_P: launch_tile_mode<T, PASS_RESID_P>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_SPMV_DOT: launch_tile_mode<T, PASS_SPMV_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            case PASS_POWER: launch_tile_mode<T, PASS_POWER>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
            default: throw Error(-1, "bad pass mode");
        }
        return;
    }
    switch (mode) {
        case PASS_JACOBI: launch_pass_mode<T, PASS_JACOBI>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case PASS_JACOBI_DOT: launch_pass_mode<T, PASS_JACOBI_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case PASS_RESID_P: launch_pass_mode<T, PASS_RESID_P>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case PASS_SPMV_DOT: launch_pass_mode<T, PASS_SPMV_DOT>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        case PASS_POWER: launch_pass_mode<T, PASS_POWER>(A, x, b, y, aux, omega, alpha, xprev, parts, parts2, s); break;
        default: throw Error(-1, "bad pass mode");
    }
}

template <class T>
void vec_jacobi0(int32_t n, const T* dinv, const T* b, double omega, T* y, cudaStream_t s) {
    if (!n) return;
    if (al16(dinv) && al16(b) && al16(y))
        k_jacobi0<T, true><<<chunk_grid<T, true>(n), PB, 0, s>>>(n, dinv, b, omega, y);
    else
        k_jacobi0<T, false><<<chunk_grid<T, false>(n), PB, 0, s>>>(n, dinv, b, omega, y);
    MG_LAUNCH_CHECK();
}
template <class T>
void restrict_members(int32_t nc, const int64_t* mptr, const int32_t* mlist, const T* t, T* bc, cudaStream_t s) {
    if (!nc) return;
    // 16 lanes per aggregate, 4 member loads in flight per lane (tools/ab_frames.py on hierarchy B: 68.27 ms/frame
    // with 8 x 4, 67.91 with 16 x 4; 4 x 4/8, 8 x 8, 16 x 2, 32 x 2/4 between or slower); MGPBD_RESTRICT_G8=1: 8 x 4
    const bool g8 = std::getenv("MGPBD_RESTRICT_G8") != nullptr;
    const int g = (int)std::min<int64_t>(((int64_t)nc * (g8 ? 8 : 16) * 4 + PB - 1) / PB, 148 * 8);
    if (g8) k_restrict<T, 8, 4><<<g, PB, 0, s>>>(nc, mptr, mlist, t, bc);
    else k_restrict<T, 16, 4><<<g, PB, 0, s>>>(nc, mptr, mlist, t, bc);
    MG_LAUNCH_CHECK();
}
template <class T>
void prolong_add(int32_t n, const int32_t* agg, const T* P, const T* e, T* x, cudaStream_t s) {
    if (!n) return;
    if (al16(agg) && al16(P) && al16(x))
        k_prolong<T, true><<<chunk_grid<T, true>(n), PB, 0, s>>>(n, agg, P, e, x);
    else
        k_prolong<T, false><<<chunk_grid<T, false>(n), PB, 0, s>>>(n, agg, P, e, x);
    MG_LAUNCH_CHECK();
}
template <class T>
void gs_sweep(const Csr<T>& A, const int64_t* gs_ptr, const int32_t* gs_list, int ncol, bool backward, const T* b, T* x,
              cudaStream_t s) {
    for (int t = 0; t < ncol; ++t) {
        const int c = backward ? ncol - 1 - t : t;
        k_gs_colour_smooth<T><<<148 * 4, PB, 0, s>>>(A.rowptr, A.col, A.val, gs_ptr, gs_list, c, b, x);
        MG_LAUNCH_CHECK();
    }
}
template <class T>
void pcg_update_p(int32_t n, const T* z, T* p, const double* scal, int k, cudaStream_t s) {
    if (!n) return;
    k_pcg_p<T><<<vgrid(n), PB, 0, s>>>(n, z, p, scal, k);
    MG_LAUNCH_CHECK();
}
template <class T>
void pcg_update_p_fin(int32_t n, const T* z, T* p, double* scal, int k, const double* prz, const double* prr, int np,
                      int* flags, int tag, cudaStream_t s, const double* fin) {
    // every CTA must run (CTA 0 publishes the scalars even for n = 0): the grid covers at least one chunk
    const int cpt = vec_cpt();
    if (al16(z) && al16(p)) {
#define MG_PF(C) k_pcg_p_fin<T, true, C><<<chunk_grid<T, true>(n, C), PB, 0, s>>>(n, z, p, scal, k, prz, prr, np, flags, tag, fin)
        switch (cpt) { case 1: MG_PF(1); break; case 2: MG_PF(2); break; case 8: MG_PF(8); break; default: MG_PF(4); }
#undef MG_PF
    } else {
        k_pcg_p_fin<T, false, 1><<<chunk_grid<T, false>(n), PB, 0, s>>>(n, z, p, scal, k, prz, prr, np, flags, tag, fin);
    }
    MG_LAUNCH_CHECK();
}
template <class T>
void pcg_update_xr_fin(int32_t n, const T* p, const T* q, T* x, T* r, double* scal, int k, const double* ppq, int np,
                       int* flags, int tag, cudaStream_t s, const T* dinv, double om0, T* x1, const double* fin) {
    const int cpt = vec_cpt();
    if (al16(p) && al16(q) && al16(x) && al16(r) && (!x1 || (al16(x1) && al16(dinv)))) {
#define MG_XR(C) k_pcg_xr_fin<T, true, C><<<chunk_grid<T, true>(n, C), PB, 0, s>>>(n, p, q, x, r, scal, k, ppq, np, flags, tag, dinv, om0, x1, fin)
        switch (cpt) { case 1: MG_XR(1); break; case 2: MG_XR(2); break; case 8: MG_XR(8); break; default: MG_XR(4); }
#undef MG_XR
    } else {
        k_pcg_xr_fin<T, false, 1><<<chunk_grid<T, false>(n), PB, 0, s>>>(n, p, q, x, r, scal, k, ppq, np, flags, tag, dinv, om0, x1, fin);
    }
    MG_LAUNCH_CHECK();
}
template <class T>
void pcg_update_xr(int32_t n, const T* p, const T* q, T* x, T* r, const double* scal, int k, cudaStream_t s) {
    if (!n) return;
    k_pcg_xr<T><<<vgrid(n), PB, 0, s>>>(n, p, q, x, r, scal, k);
    MG_LAUNCH_CHECK();
}
template <class T>
void dot_parts(int32_t n, const T* a, const T* b, double* parts, int grid, cudaStream_t s) {
    k_dot<T><<<grid, PB, 0, s>>>(n, a, b, parts);
    MG_LAUNCH_CHECK();
}
template <class T>
void scale_by_inv_sqrt(int32_t n, const T* w, T* v, const double* ss, cudaStream_t s) {
    if (!n) return;
    k_scale<T><<<vgrid(n), PB, 0, s>>>(n, w, v, ss);
    MG_LAUNCH_CHECK();
}
void pcg_finalize_rz(const double* prz, const double* prr, int np, double* scal, int k, int* flags, int tag,
                     cudaStream_t s) {
    k_fin_rz<<<1, 1024, 0, s>>>(prz, prr, np, scal, k, flags, tag);
    MG_LAUNCH_CHECK();
}
void pcg_finalize_pq(const double* p, int np, double* scal, int k, int* flags, int tag, cudaStream_t s) {
    k_fin_pq<<<1, 1024, 0, s>>>(p, np, scal, k, flags, tag);
    MG_LAUNCH_CHECK();
}
template <class T>
void coarse_invert(const Csr<T>& A, double* work, double* Ainv, int* flags, cudaStream_t s) {
    const int32_t n = A.n;
    size_t bytes = (size_t)n * n * sizeof(double);
    // n >= MGPBD_GJ_BIG_N (default 1024): the 3-kernel panel loop with the register-tiled update (k_gj_update64)
    const char* bn = std::getenv("MGPBD_GJ_BIG_N");
    const bool big = n >= (bn ? std::atoi(bn) : 1024);
    const bool coop = std::getenv("MGPBD_NO_GJ_COOP") == nullptr && !big;
    // (the one-CTA scalar Gauss-Jordan in shared memory is n barrier-separated steps: 241 us at n = 102
    // against ~40 us for the cooperative blocked kernel, so it only serves as the MGPBD_NO_GJ_COOP path)
    if (!coop && !big && bytes <= 160 * 1024) {  // small: whole matrix in one CTA's shared memory
        if (bytes > 48 * 1024)
            ensure_dyn_smem((const void*)k_coarse_inv<T>, bytes);
        k_coarse_inv<T><<<1, 1024, bytes, s>>>(n, A.rowptr, A.col, A.val, work, Ainv, flags, 1);
        MG_LAUNCH_CHECK();
        return;
    }
    if (coop) {  // one cooperative launch; work is the second n x n buffer
        static const int grid = [] {  // thread-safe one-time initialisation
            int dev = 0, sms = 0, occ = 0;
            MG_CK(cudaGetDevice(&dev));
            MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gj_coop<T>, GJT, 0));
            return sms * std::max(1, std::min(occ, 2));
        }();
        const int npan = (n + 31) / 32;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(std::min(grid, npan * npan));
        cfg.blockDim = dim3(GJT);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MG_CK(cudaLaunchKernelEx(&cfg, k_gj_coop<T>, n, A.rowptr, A.col, A.val, Ainv, work, flags));
        MG_LAUNCH_CHECK();
        return;
    }
    // blocked Gauss-Jordan in place on Ainv; work holds P (GJB^2), C (n*GJB), R (GJB*n)
    double* P = work;
    double* Cb = work + GJB * GJB;
    double* Rb = Cb + (size_t)n * GJB;
    k_dense_load<T><<<(int)std::min<int64_t>(((int64_t)n * 32 + 255) / 256, 148 * 8), 256, 0, s>>>(n, A.rowptr, A.col,
                                                                                                   A.val, Ainv);
    MG_LAUNCH_CHECK();
    const dim3 ug((n + 31) / 32, (n + 31) / 32);
    for (int32_t k0 = 0; k0 < n; k0 += GJB) {
        const int32_t bs = std::min<int32_t>(GJB, n - k0);
        k_gj_diag<<<1, 1024, 0, s>>>(n, Ainv, k0, bs, P, flags);
        MG_LAUNCH_CHECK();
        k_gj_panel<<<(int)std::min<int64_t>((2 * (int64_t)n * bs + 255) / 256, 148 * 8), 256, 0, s>>>(n, Ainv, k0, bs, P,
                                                                                                   Cb, Rb);
        MG_LAUNCH_CHECK();
        if (big) k_gj_update64<<<dim3((n + 63) / 64, (n + 63) / 64), GJU_T, 0, s>>>(n, Ainv, k0, bs, P, Cb, Rb);
        else k_gj_update<<<ug, 256, 0, s>>>(n, Ainv, k0, bs, P, Cb, Rb);
        MG_LAUNCH_CHECK();
    }
}
template <class T>
void coarse_gemv(int32_t n, const double* Ainv, const T* b, T* x, cudaStream_t s) {
    if (!n) return;
    int g = (int)std::min<int64_t>(((int64_t)n * 32 + PB - 1) / PB, 148 * 8);
    k_coarse_gemv<T><<<g, PB, 0, s>>>(n, Ainv, b, x);
    MG_LAUNCH_CHECK();
}

#define MG_INST(T)                                                                                            \
    template void csr_pass<T>(int, const Csr<T>&, const T*, const T*, T*, const T*, double, double*, double*,  \
                              cudaStream_t, double, const T*);                                                 \
    template void vec_jacobi0<T>(int32_t, const T*, const T*, double, T*, cudaStream_t);                       \
    template void restrict_members<T>(int32_t, const int64_t*, const int32_t*, const T*, T*, cudaStream_t);    \
    template void prolong_add<T>(int32_t, const int32_t*, const T*, const T*, T*, cudaStream_t);               \
    template void pcg_update_p<T>(int32_t, const T*, T*, const double*, int, cudaStream_t);                    \
    template void gs_sweep<T>(const Csr<T>&, const int64_t*, const int32_t*, int, bool, const T*, T*, cudaStream_t); \
    template void pcg_update_xr<T>(int32_t, const T*, const T*, T*, T*, const double*, int, cudaStream_t);     \
    template void pcg_update_p_fin<T>(int32_t, const T*, T*, double*, int, const double*, const double*, int,  \
                                      int*, int, cudaStream_t, const double*);                                \
    template void pcg_update_xr_fin<T>(int32_t, const T*, const T*, T*, T*, double*, int, const double*, int,  \
                                       int*, int, cudaStream_t, const T*, double, T*, const double*);         \
    template void dot_parts<T>(int32_t, const T*, const T*, double*, int, cudaStream_t);                       \
    template void scale_by_inv_sqrt<T>(int32_t, const T*, T*, const double*, cudaStream_t);                    \
    template void coarse_invert<T>(const Csr<T>&, double*, double*, int*, cudaStream_t);                       \
    template void coarse_gemv<T>(int32_t, const double*, const T*, T*, cudaStream_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
