// AMG setup kernels and the Galerkin product (see setup.cuh).
#include <climits>
#include <cstdlib>
#include <cooperative_groups.h>

#include "setup.cuh"
#include "util.cuh"

namespace cg = cooperative_groups;

namespace mgpbd {
namespace {

inline int g1(int64_t n, int bs = 256) {
    int64_t g = (n + bs - 1) / bs;
    return (int)(g > 0 ? g : 1);
}
inline int gw(int64_t nrows, int bs = 256) {  // warp per row
    int64_t g = (nrows * 32 + bs - 1) / bs;
    if (g < 1) g = 1;
    return (int)(g < 148 * 16 ? g : 148 * 16);
}

__device__ __forceinline__ bool prio_less(uint64_t ka, int32_t a, uint64_t kb, int32_t b) {
    return ka < kb || (ka == kb && a < b);
}

// ----------------------------------------------------------------------------- SOC
__global__ void k_soc(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                      const double* __restrict__ val, double theta, uint8_t* __restrict__ strong) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        const double aii = fabs(val[e1 - 1]);
        for (int64_t e = e0 + lane; e < e1; e += 32) {
            const int32_t j = col[e];
            uint8_t st = 0;
            if (j != i) {
                const double ajj = fabs(val[rowptr[j + 1] - 1]);
                st = fabs(val[e]) >= theta * sqrt(aii * ajj) ? 1 : 0;
            }
            strong[e] = st;
        }
    }
}

// ----------------------------------------------------------------------------- aggregation
__global__ void k_keys(int32_t n, uint64_t base, uint64_t* __restrict__ keys) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) keys[i] = hkey(base, (uint64_t)i);
}

// m1[i] = highest-priority undecided node in the closed strong neighbourhood of i (-1 if none)
__global__ void k_min1(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const uint8_t* __restrict__ strong, const int8_t* __restrict__ state,
                       const uint64_t* __restrict__ keys, int32_t* __restrict__ m1) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t best = -1;
    uint64_t bk = 0;
    if (state[i] == 0) { best = i; bk = keys[i]; }
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        if (!strong[e]) continue;
        int32_t j = col[e];
        if (state[j] != 0) continue;
        uint64_t kj = keys[j];
        if (best < 0 || prio_less(kj, j, bk, best)) { best = j; bk = kj; }
    }
    m1[i] = best;
}

// undecided i joins the MIS of S^2 iff it is the highest-priority undecided node within distance 2
__global__ void k_min2(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const uint8_t* __restrict__ strong, int8_t* __restrict__ state,
                       const uint64_t* __restrict__ keys, const int32_t* __restrict__ m1, uint8_t* __restrict__ newseed) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || state[i] != 0) return;
    int32_t best = m1[i];
    uint64_t bk = keys[best];
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        if (!strong[e]) continue;
        int32_t c = m1[col[e]];
        if (c < 0) continue;
        uint64_t kc = keys[c];
        if (prio_less(kc, c, bk, best)) { best = c; bk = kc; }
    }
    if (best == i) { state[i] = 1; newseed[i] = 1; }
}

__global__ void k_mark1(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const uint8_t* __restrict__ strong, const uint8_t* __restrict__ newseed, uint8_t* __restrict__ f1) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t f = newseed[i];
    for (int64_t e = rowptr[i]; e < rowptr[i + 1] && !f; ++e)
        if (strong[e] && newseed[col[e]]) f = 1;
    f1[i] = f;
}

__global__ void k_mark2(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const uint8_t* __restrict__ strong, const uint8_t* __restrict__ f1, int8_t* __restrict__ state,
                        int32_t* __restrict__ undecided) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || state[i] != 0) return;
    bool out = f1[i];
    for (int64_t e = rowptr[i]; e < rowptr[i + 1] && !out; ++e)
        if (strong[e] && f1[col[e]]) out = true;
    if (out) state[i] = 2;
    else atomicAdd(undecided, 1);
}

__global__ void k_lab(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                      const uint8_t* __restrict__ strong, const int8_t* __restrict__ state, int32_t* __restrict__ lab,
                      int32_t* __restrict__ seedflag) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t l = -1;
    if (state[i] == 1) l = i;
    else
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (strong[e] && state[col[e]] == 1) { l = col[e]; break; }
    lab[i] = l;
    seedflag[i] = state[i] == 1 ? 1 : 0;
}

__global__ void k_p1(int32_t n, const int32_t* __restrict__ lab, const int64_t* __restrict__ sid, int32_t* __restrict__ p1) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t l = lab[i];
    p1[i] = l >= 0 ? (int32_t)sid[l] : -1;
}

// leftovers join the pass-1 aggregate of their strongest strong neighbour; ties -> lowest id
__global__ void k_pass2(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const double* __restrict__ val, const uint8_t* __restrict__ strong,
                        const int32_t* __restrict__ p1, int32_t* __restrict__ agg, int32_t* __restrict__ orphan) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t a = p1[i];
    if (a < 0) {
        double best = -1.0;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            if (!strong[e]) continue;
            int32_t c = p1[col[e]];
            if (c < 0) continue;
            double s = fabs(val[e]);
            if (s > best || (s == best && c < a)) { best = s; a = c; }
        }
        if (a < 0) atomicExch(orphan, 1);
    }
    agg[i] = a;
}

// ----------------------------------------------------------------------------- colouring
__global__ void k_colour_round(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                               const uint64_t* __restrict__ keys, int32_t* colours, int32_t* remaining,
                               int32_t* overflow) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || colours[i] >= 0) return;
    const uint64_t ki = keys[i];
    uint64_t used[4] = {0, 0, 0, 0};
    bool ready = true;
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        int32_t j = col[e];
        if (j == i || !prio_less(keys[j], j, ki, i)) continue;
        int32_t c = *(volatile int32_t*)&colours[j];
        if (c < 0) { ready = false; break; }
        if (c < 256) used[c >> 6] |= 1ull << (c & 63);
    }
    if (!ready) { atomicAdd(remaining, 1); return; }
    int32_t c = 256;
    for (int w = 0; w < 4; ++w)
        if (~used[w]) { c = w * 64 + __ffsll((long long)~used[w]) - 1; break; }
    if (c >= 256) { atomicExch(overflow, 1); c = 255; }
    colours[i] = c;
}
__global__ void k_max_i32(int32_t n, const int32_t* __restrict__ v, int32_t* out) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMax(out, v[i]);
}

// ----------------------------------------------------------------------------- GS bootstrap
__global__ void k_absmax_parts(int64_t nnz, const double* __restrict__ val, double* parts) {
    double v = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        v = fmax(v, fabs(val[e]));
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) parts[blockIdx.x] = v;
    }
}
__global__ void k_gs_init(int32_t n, uint64_t base, uint64_t off, const double* __restrict__ maxabs, double* __restrict__ x) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = hunit(hkey(base, (uint64_t)i + off)) * (*maxabs);
}
// one colour class of a GS sweep on A x = 0: x_i = -(sum_{j != i} A_ij x_j) / A_ii
__global__ void k_gs_colour(int64_t cnt, const int32_t* __restrict__ rows, const int64_t* __restrict__ rowptr,
                            const int32_t* __restrict__ col, const double* __restrict__ val, double* __restrict__ x) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < cnt; t += nw) {
        const int32_t i = rows[t];
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1] - 1;
        double s = 0.0;
        for (int64_t e = e0 + lane; e < e1; e += 32) s += val[e] * x[col[e]];
        s = group_sum<32>(s);
        if (lane == 0) x[i] = -s / val[e1];
    }
}
// u_v = sum over v's incidences (constraint j, slot s) of h_{j,s} x_j (fp64, incidence order)
__global__ void k_gs_u(int32_t nv, const int64_t* __restrict__ vptr, const int32_t* __restrict__ vlist, int kc,
                       const double* __restrict__ h, const double* __restrict__ x, double* __restrict__ u) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int64_t e = vptr[v]; e < vptr[v + 1]; ++e) {
            const int32_t code = vlist[e];
            const double xj = x[code / kc];
            a += h[(int64_t)code * 3] * xj;
            b += h[(int64_t)code * 3 + 1] * xj;
            c += h[(int64_t)code * 3 + 2] * xj;
        }
        u[3 * (int64_t)v] = a; u[3 * (int64_t)v + 1] = b; u[3 * (int64_t)v + 2] = c;
    }
}
// one colour of a matrix-free GS sweep (b = 0), thread per row
template <int KC>
__global__ void k_gs_colour_mf(int64_t cnt, const int32_t* __restrict__ rows, const int32_t* __restrict__ verts,
                               const double* __restrict__ h, const double* __restrict__ at,
                               const double* __restrict__ dinv, double* __restrict__ x, double* __restrict__ u) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cnt; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = rows[t];
        int32_t v[KC];
        double hh[KC][3];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            v[k] = verts[(int64_t)i * KC + k];
#pragma unroll
            for (int d = 0; d < 3; ++d) hh[k][d] = h[((int64_t)i * KC + k) * 3 + d];
        }
        const double xi = x[i];
        double ax = at[i] * xi;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const double* uv = u + 3 * (int64_t)v[k];
            ax += hh[k][0] * uv[0] + hh[k][1] * uv[1] + hh[k][2] * uv[2];
        }
        const double dx = -ax * dinv[i];
        x[i] = xi + dx;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            double* uv = u + 3 * (int64_t)v[k];
            uv[0] += hh[k][0] * dx; uv[1] += hh[k][1] * dx; uv[2] += hh[k][2] * dx;
        }
    }
}
__global__ void k_fill_d(int32_t n, double* x, double v) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

// ----------------------------------------------------------------------------- prolongator
__global__ void k_prolongator(int32_t na, const int64_t* __restrict__ mptr, const int32_t* __restrict__ mlist,
                              const double* __restrict__ B, double* __restrict__ P, double* __restrict__ Bn) {
    int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= na) return;
    const int64_t b = mptr[a], e = mptr[a + 1];
    double ss = 0.0;
    for (int64_t k = b; k < e; ++k) { double v = B[mlist[k]]; ss += v * v; }
    const double nrm = sqrt(ss);
    Bn[a] = nrm;
    const double uni = 1.0 / sqrt((double)(e - b));
    for (int64_t k = b; k < e; ++k) { int32_t i = mlist[k]; P[i] = nrm > 0.0 ? B[i] / nrm : uni; }
}

// ----------------------------------------------------------------------------- Galerkin symbolic
__global__ void k_rowlen_max(int32_t n, const int64_t* __restrict__ rowptr, int32_t* out) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMax(out, (int32_t)(rowptr[i + 1] - rowptr[i]));
}

// warp per fine row: rank entries by (agg(col), col) -> gperm; count distinct aggregates
__global__ void k_gsort(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const int32_t* __restrict__ agg, int maxlen, uint16_t* __restrict__ gperm,
                        int32_t* __restrict__ nseg) {
    extern __shared__ uint64_t skey[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* key = skey + (int64_t)warp * maxlen;
    const int wpb = blockDim.x >> 5;
    for (int64_t i = (int64_t)blockIdx.x * wpb + warp; i < n; i += (int64_t)gridDim.x * wpb) {
        const int64_t e0 = rowptr[i];
        const int L = (int)(rowptr[i + 1] - e0);
        for (int k = lane; k < L; k += 32) {
            int32_t c = col[e0 + k];
            key[k] = ((uint64_t)(uint32_t)agg[c] << 32) | (uint32_t)c;
        }
        __syncwarp();
        int heads = 0;
        for (int k = lane; k < L; k += 32) {
            const uint64_t kk = key[k];
            int r = 0;
            bool head = true;
            for (int q = 0; q < L; ++q) {
                uint64_t kq = key[q];
                r += kq < kk;
                if ((kq >> 32) == (kk >> 32) && kq < kk) head = false;
            }
            gperm[e0 + r] = (uint16_t)k;
            heads += head;
        }
        for (int o = 16; o > 0; o >>= 1) heads += __shfl_xor_sync(0xffffffffu, heads, o);
        if (lane == 0) nseg[i] = heads;
        __syncwarp();
    }
}

// warp per fine row: write the segment table (tstart, trow, tagg)
__global__ void k_tfill(int32_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const int32_t* __restrict__ agg, const uint16_t* __restrict__ gperm,
                        const int64_t* __restrict__ tptr, int64_t* __restrict__ tstart, int32_t* __restrict__ trow,
                        int32_t* __restrict__ tagg) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        const int64_t e0 = rowptr[i];
        const int L = (int)(rowptr[i + 1] - e0);
        int64_t base = tptr[i];
        for (int q0 = 0; q0 < L; q0 += 32) {
            const int q = q0 + lane;
            int32_t a = -1, ap = -1;
            if (q < L) {
                a = agg[col[e0 + gperm[e0 + q]]];
                if (q > 0) ap = agg[col[e0 + gperm[e0 + q - 1]]];
            }
            const bool head = q < L && (q == 0 || a != ap);
            const unsigned bal = __ballot_sync(0xffffffffu, head);
            if (head) {
                int64_t t = base + __popc(bal & ((1u << lane) - 1u));
                tstart[t] = e0 + q;
                trow[t] = (int32_t)i;
                tagg[t] = a;
            }
            base += __popc(bal);
        }
    }
}

__global__ void k_cand_count(int32_t na, const int64_t* __restrict__ mptr, const int32_t* __restrict__ mlist,
                             const int64_t* __restrict__ tptr, int32_t* out_max) {
    int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= na) return;
    int64_t c = 0;
    for (int64_t k = mptr[a]; k < mptr[a + 1]; ++k) { int32_t i = mlist[k]; c += tptr[i + 1] - tptr[i]; }
    atomicMax(out_max, (int32_t)(c < INT_MAX ? c : INT_MAX));
}

// warp per coarse row: unique sorted coarse columns of the row (MODE 0 count, MODE 1 fill)
template <int MODE>
__global__ void k_crow(int32_t na, const int64_t* __restrict__ mptr, const int32_t* __restrict__ mlist,
                       const int64_t* __restrict__ tptr, const int32_t* __restrict__ tagg, int maxc,
                       int32_t* __restrict__ ccnt, const int64_t* __restrict__ crowptr, int32_t* __restrict__ ccol) {
    extern __shared__ int32_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t* cand = sm + (int64_t)warp * 2 * maxc;
    int32_t* first = cand + maxc;
    const int wpb = blockDim.x >> 5;
    for (int64_t a = (int64_t)blockIdx.x * wpb + warp; a < na; a += (int64_t)gridDim.x * wpb) {
        // gather candidates
        int C = 0;
        for (int64_t k = mptr[a]; k < mptr[a + 1]; ++k) {
            int32_t i = mlist[k];
            const int64_t t0 = tptr[i], t1 = tptr[i + 1];
            for (int64_t t = t0 + lane; t < t1; t += 32) {
                int32_t b = tagg[t];
                cand[C + (t - t0)] = (b == a) ? INT_MAX : b;
            }
            C += (int)(t1 - t0);
        }
        __syncwarp();
        for (int p = lane; p < C; p += 32) {
            int32_t v = cand[p];
            int f = v != INT_MAX;
            for (int q = 0; q < p && f; ++q) f = cand[q] != v;
            first[p] = f;
        }
        __syncwarp();
        if (MODE == 0) {
            int c = 0;
            for (int p = lane; p < C; p += 32) c += first[p];
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) ccnt[a] = c + 1;
        } else {
            const int64_t base = crowptr[a];
            for (int p = lane; p < C; p += 32) {
                if (!first[p]) continue;
                int32_t v = cand[p];
                int r = 0;
                for (int q = 0; q < C; ++q) r += (first[q] && cand[q] < v);
                ccol[base + r] = v;
            }
            if (lane == 0) ccol[crowptr[a + 1] - 1] = (int32_t)a;
        }
        __syncwarp();
    }
}

// coarse nnz index of each segment
__global__ void k_cidx(int64_t T, const int32_t* __restrict__ trow, const int32_t* __restrict__ tagg,
                       const int32_t* __restrict__ agg, const int64_t* __restrict__ crowptr,
                       const int32_t* __restrict__ ccol, int32_t* __restrict__ cidx) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const int32_t a = agg[trow[t]], b = tagg[t];
    const int64_t r0 = crowptr[a], r1 = crowptr[a + 1] - 1;
    int64_t pos = r1;
    if (b != a) {
        int64_t lo = r0, hi = r1;  // search in [r0, r1)
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (ccol[mid] < b) lo = mid + 1; else hi = mid;
        }
        pos = lo;
    }
    cidx[t] = (int32_t)pos;
}

// ----------------------------------------------------------------------------- Galerkin numeric
template <class T>
__global__ void k_gal1(int64_t T_, const int64_t* __restrict__ tstart, const int32_t* __restrict__ trow,
                       const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const uint16_t* __restrict__ gperm, const T* __restrict__ val, const T* __restrict__ P,
                       T* __restrict__ tval) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T_) return;
    const int32_t i = trow[t];
    const int64_t e0 = rowptr[i];
    double s = 0.0;
    for (int64_t q = tstart[t]; q < tstart[t + 1]; ++q) {
        const int64_t e = e0 + gperm[q];
        s += (double)val[e] * (double)P[col[e]];
    }
    tval[t] = (T)((double)P[i] * s);
}
template <class T>
__global__ void k_gal2(int64_t cnnz, const int64_t* __restrict__ lptr, const int32_t* __restrict__ llist,
                       const T* __restrict__ tval, T* __restrict__ cval) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= cnnz) return;
    double s = 0.0;
    for (int64_t k = lptr[c]; k < lptr[c + 1]; ++k) s += (double)tval[llist[k]];
    cval[c] = (T)s;
}
template <class T>
__global__ void k_diag_inv(int32_t n, const int64_t* __restrict__ rowptr, const T* __restrict__ val, T* __restrict__ dinv) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dinv[i] = (T)(1.0 / (double)val[rowptr[i + 1] - 1]);
}

__global__ void k_power_init(int32_t n, uint64_t base, double* v) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = hunit(hkey(base, (uint64_t)i));
}

}  // namespace

void soc(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, double theta, uint8_t* strong,
         cudaStream_t s) {
    if (!n) return;
    k_soc<<<gw(n), 256, 0, s>>>(n, rowptr, col, val, theta, strong);
    MG_LAUNCH_CHECK();
}

int32_t aggregate(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, const uint8_t* strong,
                  uint64_t seed, int level, int32_t* agg, cudaStream_t s) {
    DBuf<uint64_t> keys; DBuf<int8_t> state; DBuf<int32_t> m1, lab, seedflag, p1, cnt;
    DBuf<uint8_t> newseed, f1; DBuf<int64_t> sid;
    keys.resize(n); state.resize(n); m1.resize(n); lab.resize(n); seedflag.resize(n); p1.resize(n);
    newseed.resize(n); f1.resize(n); sid.resize((size_t)n + 1); cnt.resize(2);
    k_keys<<<g1(n), 256, 0, s>>>(n, hkey_base(seed, 1, level), keys.p);
    MG_LAUNCH_CHECK();
    MG_CK(cudaMemsetAsync(state.p, 0, n, s));
    for (int round = 0;; ++round) {
        if (round > n + 1) throw Error(-2, "aggregation rounds did not terminate");
        MG_CK(cudaMemsetAsync(newseed.p, 0, n, s));
        MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t), s));
        k_min1<<<g1(n), 256, 0, s>>>(n, rowptr, col, strong, state.p, keys.p, m1.p);
        MG_LAUNCH_CHECK();
        k_min2<<<g1(n), 256, 0, s>>>(n, rowptr, col, strong, state.p, keys.p, m1.p, newseed.p);
        MG_LAUNCH_CHECK();
        k_mark1<<<g1(n), 256, 0, s>>>(n, rowptr, col, strong, newseed.p, f1.p);
        MG_LAUNCH_CHECK();
        k_mark2<<<g1(n), 256, 0, s>>>(n, rowptr, col, strong, f1.p, state.p, cnt.p);
        MG_LAUNCH_CHECK();
        if (read_scalar(cnt.p, s) == 0) break;
    }
    k_lab<<<g1(n), 256, 0, s>>>(n, rowptr, col, strong, state.p, lab.p, seedflag.p);
    MG_LAUNCH_CHECK();
    scan_exclusive<int32_t>(seedflag.p, sid.p, n, s);
    int32_t n_agg = (int32_t)read_scalar(sid.p + n, s);
    k_p1<<<g1(n), 256, 0, s>>>(n, lab.p, sid.p, p1.p);
    MG_LAUNCH_CHECK();
    MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t), s));
    k_pass2<<<g1(n), 256, 0, s>>>(n, rowptr, col, val, strong, p1.p, agg, cnt.p);
    MG_LAUNCH_CHECK();
    if (read_scalar(cnt.p, s) != 0) throw Error(-2, "aggregation left an unassigned node");
    return n_agg;
}

int32_t colour(int32_t n, const int64_t* rowptr, const int32_t* col, uint64_t seed, int32_t* colours, cudaStream_t s) {
    DBuf<uint64_t> keys; DBuf<int32_t> cnt;
    keys.resize(n); cnt.resize(3);
    k_keys<<<g1(n), 256, 0, s>>>(n, hkey_base(seed, 2, 0), keys.p);
    MG_LAUNCH_CHECK();
    fill_i32(colours, -1, n, s);
    MG_CK(cudaMemsetAsync(cnt.p, 0, 3 * sizeof(int32_t), s));
    for (int round = 0;; ++round) {
        if (round > n + 1) throw Error(-2, "colouring rounds did not terminate");
        MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t), s));
        k_colour_round<<<g1(n), 256, 0, s>>>(n, rowptr, col, keys.p, colours, cnt.p, cnt.p + 1);
        MG_LAUNCH_CHECK();
        if (read_scalar(cnt.p, s) == 0) break;
    }
    if (read_scalar(cnt.p + 1, s) != 0) throw Error(-2, "colouring needs more than 256 colours");
    MG_CK(cudaMemsetAsync(cnt.p + 2, 0, sizeof(int32_t), s));
    k_max_i32<<<g1(n), 256, 0, s>>>(n, colours, cnt.p + 2);
    MG_LAUNCH_CHECK();
    return read_scalar(cnt.p + 2, s) + 1;
}

void gs_bootstrap(int32_t n, const int64_t* rowptr, const int32_t* col, const double* val, const int32_t* colours,
                  int32_t ncolours, int32_t sweeps, uint64_t seed, double* B, cudaStream_t s, const GsOperator* op,
                  uint64_t idx_offset) {
    int64_t nnz = read_scalar(rowptr + n, s);
    DBuf<double> parts, mx;
    parts.resize(1024); mx.resize(2);
    k_absmax_parts<<<1024, 256, 0, s>>>(nnz, val, parts.p);
    MG_LAUNCH_CHECK();
    finalize_max(parts.p, 1024, mx.p, s);
    k_gs_init<<<g1(n), 256, 0, s>>>(n, hkey_base(seed, 3, 0), idx_offset, mx.p, B);
    MG_LAUNCH_CHECK();
    DBuf<int64_t> cptr; DBuf<int32_t> clist, cnt;
    group_by_key(colours, n, ncolours, cptr, clist, cnt, s, /*sort=*/false);
    std::vector<int64_t> hptr(ncolours + 1);
    d2h(hptr.data(), cptr.p, ncolours + 1, s);
    MG_CK(cudaStreamSynchronize(s));
    DBuf<double> u;
    if (op) {
        u.resize(3 * (size_t)op->nv);
        k_gs_u<<<g1(op->nv), 256, 0, s>>>(op->nv, op->vptr, op->vlist, op->kc, op->h, B, u.p);
        MG_LAUNCH_CHECK();
    }
    for (int sw = 0; sw < sweeps; ++sw)
        for (int c = 0; c < ncolours; ++c) {
            int64_t cntc = hptr[c + 1] - hptr[c];
            if (!cntc) continue;
            if (op) {
                const int g = (int)std::min<int64_t>((cntc + 127) / 128, 148 * 16);
                if (op->kc == 4)
                    k_gs_colour_mf<4><<<g, 128, 0, s>>>(cntc, clist.p + hptr[c], op->verts, op->h, op->at, op->dinv, B, u.p);
                else
                    k_gs_colour_mf<2><<<g, 128, 0, s>>>(cntc, clist.p + hptr[c], op->verts, op->h, op->at, op->dinv, B, u.p);
            } else {
                k_gs_colour<<<gw(cntc), 256, 0, s>>>(cntc, clist.p + hptr[c], rowptr, col, val, B);
            }
            MG_LAUNCH_CHECK();
        }
    dot_parts<double>(n, B, B, parts.p, 1024, s);
    finalize_sum(parts.p, 1024, mx.p + 1, s);
    double nn = read_scalar(mx.p + 1, s);
    if (!(sqrt(nn) >= 1e-14 * sqrt((double)n))) {
        k_fill_d<<<g1(n), 256, 0, s>>>(n, B, 1.0);
        MG_LAUNCH_CHECK();
    }
}

void prolongator(int32_t n_agg, const int64_t* mptr, const int32_t* mlist, const double* B, double* P, double* Bn,
                 cudaStream_t s) {
    if (!n_agg) return;
    k_prolongator<<<g1(n_agg, 128), 128, 0, s>>>(n_agg, mptr, mlist, B, P, Bn);
    MG_LAUNCH_CHECK();
}

void galerkin_symbolic(int32_t n, const int64_t* rowptr, const int32_t* col, const int32_t* agg, const int64_t* mptr,
                       const int32_t* mlist, int32_t n_agg, GalerkinPlan& plan, DBuf<int64_t>& crowptr,
                       DBuf<int32_t>& ccol, cudaStream_t s) {
    const int64_t nnz = read_scalar(rowptr + n, s);
    DBuf<int32_t> tmp;
    tmp.resize((size_t)std::max<int64_t>(n, n_agg) + 2);
    // 1. per-row sort by (agg, col)
    MG_CK(cudaMemsetAsync(tmp.p, 0, sizeof(int32_t), s));
    k_rowlen_max<<<g1(n), 256, 0, s>>>(n, rowptr, tmp.p);
    MG_LAUNCH_CHECK();
    const int maxlen = std::max(1, read_scalar(tmp.p, s));
    if (maxlen > 65535) throw Error(-7, "row too long for the Galerkin plan");
    int wpb = 4;
    while (wpb > 1 && (size_t)maxlen * 8 * wpb > 160 * 1024) wpb >>= 1;
    size_t smem = (size_t)maxlen * 8 * wpb;
    if (smem > 200 * 1024) throw Error(-7, "row too long for the Galerkin plan");
    if (smem > 48 * 1024) ensure_dyn_smem((const void*)k_gsort, smem);
    plan.gperm.resize(nnz);
    DBuf<int32_t> nseg;
    nseg.resize(n);
    int grid = (int)std::min<int64_t>(ceil_div(n, wpb), 148 * 64);
    k_gsort<<<grid, 32 * wpb, smem, s>>>(n, rowptr, col, agg, maxlen, plan.gperm.p, nseg.p);
    MG_LAUNCH_CHECK();
    plan.tptr.resize((size_t)n + 1);
    scan_exclusive<int32_t>(nseg.p, plan.tptr.p, n, s);
    plan.T = read_scalar(plan.tptr.p + n, s);
    plan.tstart.resize(plan.T + 1);
    plan.trow.resize(plan.T);
    plan.tagg.resize(plan.T);
    k_tfill<<<gw(n), 256, 0, s>>>(n, rowptr, col, agg, plan.gperm.p, plan.tptr.p, plan.tstart.p, plan.trow.p, plan.tagg.p);
    MG_LAUNCH_CHECK();
    h2d(plan.tstart.p + plan.T, &nnz, 1, s);
    // 2. coarse rows
    MG_CK(cudaMemsetAsync(tmp.p, 0, sizeof(int32_t), s));
    k_cand_count<<<g1(n_agg), 256, 0, s>>>(n_agg, mptr, mlist, plan.tptr.p, tmp.p);
    MG_LAUNCH_CHECK();
    const int maxc = std::max(1, read_scalar(tmp.p, s));
    int cw = 8;
    while (cw > 1 && (size_t)maxc * 8 * cw > 160 * 1024) cw >>= 1;
    size_t csm = (size_t)maxc * 8 * cw;
    if (csm > 200 * 1024) throw Error(-7, "coarse row candidate list too long");
    if (csm > 48 * 1024) {
        ensure_dyn_smem((const void*)k_crow<0>, csm);
        ensure_dyn_smem((const void*)k_crow<1>, csm);
    }
    DBuf<int32_t> ccnt;
    ccnt.resize(n_agg);
    int cgrid = (int)std::min<int64_t>(ceil_div(n_agg, cw), 148 * 64);
    k_crow<0><<<cgrid, 32 * cw, csm, s>>>(n_agg, mptr, mlist, plan.tptr.p, plan.tagg.p, maxc, ccnt.p, nullptr, nullptr);
    MG_LAUNCH_CHECK();
    crowptr.resize((size_t)n_agg + 1);
    scan_exclusive<int32_t>(ccnt.p, crowptr.p, n_agg, s);
    const int64_t cnnz = read_scalar(crowptr.p + n_agg, s);
    ccol.resize(cnnz);
    k_crow<1><<<cgrid, 32 * cw, csm, s>>>(n_agg, mptr, mlist, plan.tptr.p, plan.tagg.p, maxc, nullptr, crowptr.p, ccol.p);
    MG_LAUNCH_CHECK();
    // 3. stage-2 lists
    DBuf<int32_t> cidx, cnt;
    cidx.resize(plan.T);
    if (plan.T) {
        k_cidx<<<g1(plan.T), 256, 0, s>>>(plan.T, plan.trow.p, plan.tagg.p, agg, crowptr.p, ccol.p, cidx.p);
        MG_LAUNCH_CHECK();
    }
    group_by_key(cidx.p, plan.T, cnnz, plan.lptr, plan.llist, cnt, s, /*sort=*/true);
    MG_CK(cudaStreamSynchronize(s));
}

template <class T>
void galerkin_numeric(const GalerkinPlan& plan, const int64_t* rowptr, const int32_t* col, const T* val, const T* P,
                      int32_t n_agg, const int64_t* crowptr, int64_t cnnz, T* tval, T* cval, T* cdinv, cudaStream_t s,
                      int64_t t_begin, int64_t t_end) {
    if (t_end < 0) t_end = plan.T;
    if (t_end > t_begin) {
        const int64_t nt = t_end - t_begin;
        k_gal1<T><<<g1(nt), 256, 0, s>>>(nt, plan.tstart.p + t_begin, plan.trow.p + t_begin, rowptr, col,
                                        plan.gperm.p, val, P, tval + t_begin);
        MG_LAUNCH_CHECK();
    }
    if (cnnz) {
        k_gal2<T><<<g1(cnnz), 256, 0, s>>>(cnnz, plan.lptr.p, plan.llist.p, tval, cval);
        MG_LAUNCH_CHECK();
    }
    if (cdinv) diag_inv<T>(n_agg, crowptr, cval, cdinv, s);
}

template <class T>
void diag_inv(int32_t n, const int64_t* rowptr, const T* val, T* dinv, cudaStream_t s) {
    if (!n) return;
    k_diag_inv<T><<<g1(n), 256, 0, s>>>(n, rowptr, val, dinv);
    MG_LAUNCH_CHECK();
}

double power_method_op(int32_t n, int dot_grid, const std::function<int(const double*, double*, double*)>& apply,
                       int32_t iters, uint64_t seed, int level, double* v, double* w, double* parts, double* ss,
                       cudaStream_t s, bool init) {
    if (init) {
        k_power_init<<<g1(n), 256, 0, s>>>(n, hkey_base(seed, 4, level), v);
        MG_LAUNCH_CHECK();
        dot_parts<double>(n, v, v, parts, dot_grid, s);
        finalize_sum(parts, dot_grid, ss, s);
        scale_by_inv_sqrt<double>(n, v, v, ss, s);
    }
    for (int it = 0; it < iters; ++it) {
        const int np = apply(v, w, parts);
        finalize_sum(parts, np, ss, s);
        scale_by_inv_sqrt<double>(n, w, v, ss, s);
    }
    double lam2 = read_scalar(ss, s);
    return iters > 0 ? sqrt(lam2) : 0.0;
}

namespace {
// The whole power method of a coarse level in one cooperative launch: per iteration one phase computing
// w = D^-1 A v (warp per row) with per-CTA partials of |w|^2, a grid barrier, every CTA summing the
// partials in the same fixed order, v = w / |w| over its rows, a barrier.  Same arithmetic as the
// launch-per-step version (k_power_init, PASS_POWER, k_finalize_sum, k_scale); ~3 launches per
// iteration (~1.4 ms per level at 100 iterations) become ~2 barriers per iteration.
constexpr int PWT = 512;
__device__ __forceinline__ double pw_total(const double* __restrict__ parts, int np, double* sh) {
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += PWT) v += parts[i];
    return block_sum<PWT>(v, sh);
}
__global__ void __launch_bounds__(PWT) k_power_coop(int32_t n, const int64_t* __restrict__ rowptr,
                                                    const int32_t* __restrict__ col, const double* __restrict__ val,
                                                    const double* __restrict__ dinv, int32_t iters, uint64_t base,
                                                    double* __restrict__ v, double* __restrict__ w,
                                                    double* __restrict__ parts, double* __restrict__ out, int init) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[32];
    __shared__ double inv_s;
    const int lane = threadIdx.x & 31;
    const int64_t tid = (int64_t)blockIdx.x * PWT + threadIdx.x, nt = (int64_t)gridDim.x * PWT;
    const int64_t gw = tid >> 5, nw = nt >> 5;
    double acc = 0.0, t = 0.0, ss = 0.0;
    if (init) {  // v_0 = U(stream 4)/|.|
        for (int64_t i = tid; i < n; i += nt) {
            const double x = hunit(hkey(base, (uint64_t)i));
            v[i] = x;
            acc += x * x;
        }
        t = block_sum<PWT>(acc, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t;
        grid.sync();
        ss = pw_total(parts, gridDim.x, sh);
        if (threadIdx.x == 0) { const double lam = sqrt(ss); inv_s = lam > 0.0 ? 1.0 / lam : 0.0; }
        __syncthreads();
        for (int64_t i = tid; i < n; i += nt) v[i] = v[i] * inv_s;
        grid.sync();
    }
    for (int32_t it = 0; it < iters; ++it) {
        acc = 0.0;
        for (int64_t i = gw; i < n; i += nw) {
            double s = 0.0;
            for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) s += val[e] * v[col[e]];
            s = group_sum<32>(s);
            if (lane == 0) {
                const double wi = dinv[i] * s;
                w[i] = wi;
                acc += wi * wi;
            }
        }
        t = block_sum<PWT>(acc, sh);
        if (threadIdx.x == 0) parts[blockIdx.x] = t;
        grid.sync();
        ss = pw_total(parts, gridDim.x, sh);
        if (threadIdx.x == 0) { const double lam = sqrt(ss); inv_s = lam > 0.0 ? 1.0 / lam : 0.0; }
        __syncthreads();
        for (int64_t i = tid; i < n; i += nt) v[i] = w[i] * inv_s;
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = ss;
}
}  // namespace

double power_method(const Csr<double>& A, int32_t iters, uint64_t seed, int level, double* v, double* w,
                    double* parts, double* ss, cudaStream_t s, bool init) {
    if (A.n > 0 && A.n <= (1 << 18) && std::getenv("MGPBD_NO_POWER_COOP") == nullptr) {
        static const int grid = [] {
            int dev = 0, sms = 0, occ = 0;
            MG_CK(cudaGetDevice(&dev));
            MG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            MG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_power_coop, PWT, 0));
            return sms * std::max(1, std::min(occ, 2));
        }();
        // parts holds >= 1024 doubles (the engine's partial-sum buffer)
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(grid, 1024), ((int64_t)A.n * 32 + PWT - 1) / PWT));
        const uint64_t base = hkey_base(seed, 4, level);
        int init_i = init ? 1 : 0;
        void* args[] = {(void*)&A.n, (void*)&A.rowptr, (void*)&A.col, (void*)&A.val, (void*)&A.dinv,
                        (void*)&iters, (void*)&base, (void*)&v, (void*)&w, (void*)&parts, (void*)&ss, (void*)&init_i};
        MG_CK(cudaLaunchCooperativeKernel((const void*)k_power_coop, g, PWT, args, 0, s));
        MG_LAUNCH_CHECK();
        const double lam2 = read_scalar(ss, s);
        return iters > 0 ? sqrt(lam2) : 0.0;
    }
    return power_method_op(
        A.n, A.grid,
        [&](const double* x, double* y, double* pp) {
            csr_pass<double>(PASS_POWER, A, x, nullptr, y, nullptr, 0.0, pp, nullptr, s);
            return A.nparts;
        },
        iters, seed, level, v, w, parts, ss, s, init);
}

#define MG_INST(T)                                                                                             \
    template void galerkin_numeric<T>(const GalerkinPlan&, const int64_t*, const int32_t*, const T*, const T*,  \
                                      int32_t, const int64_t*, int64_t, T*, T*, T*, cudaStream_t, int64_t,     \
                                      int64_t);                                                                \
    template void diag_inv<T>(int32_t, const int64_t*, const T*, T*, cudaStream_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
