// Constraint-side kernels of the MGPBD hot path (see mesh.cuh).
#include <climits>
#include <type_traits>

#include "mesh.cuh"
#include "record.cuh"
#include "util.cuh"

namespace mgpbd {
namespace {

inline int grid1d(int64_t n, int bs = 256) {
    int64_t g = (n + bs - 1) / bs;
    return (int)(g > 0 ? g : 1);
}

// ----------------------------------------------------------------------------- rest data
__global__ void k_rest_distance(const int32_t* __restrict__ verts, const double* __restrict__ X, int32_t m,
                                double* __restrict__ L) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    int a = verts[2 * j], b = verts[2 * j + 1];
    double d0 = X[3 * a] - X[3 * b], d1 = X[3 * a + 1] - X[3 * b + 1], d2 = X[3 * a + 2] - X[3 * b + 2];
    L[j] = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

// D_m (columns X_k - X_0), its inverse (row-major 9), V = |det D_m|/6.
__global__ void k_rest_arap(const int32_t* __restrict__ verts, const double* __restrict__ X, int32_t m,
                            double* __restrict__ Dminv, double* __restrict__ vol, int32_t* bad) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int* tv = verts + 4 * (int64_t)j;
    double D[9];
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) D[r * 3 + c] = X[3 * tv[1 + c] + r] - X[3 * tv[0] + r];
    double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[5] * D[6] - D[3] * D[8], c02 = D[3] * D[7] - D[4] * D[6];
    double det = D[0] * c00 + D[1] * c01 + D[2] * c02;
    vol[j] = fabs(det) / 6.0;
    double* Di = Dminv + 9 * (int64_t)j;
    if (det == 0.0) {
        for (int k = 0; k < 9; ++k) Di[k] = 0.0;
        atomicExch(bad, 1);
        return;
    }
    double id = 1.0 / det;
    Di[0] = c00 * id;
    Di[1] = (D[2] * D[7] - D[1] * D[8]) * id;
    Di[2] = (D[1] * D[5] - D[2] * D[4]) * id;
    Di[3] = c01 * id;
    Di[4] = (D[0] * D[8] - D[2] * D[6]) * id;
    Di[5] = (D[2] * D[3] - D[0] * D[5]) * id;
    Di[6] = c02 * id;
    Di[7] = (D[1] * D[6] - D[0] * D[7]) * id;
    Di[8] = (D[0] * D[4] - D[1] * D[3]) * id;
}

// ----------------------------------------------------------------------------- incidence
__global__ void k_count_inc(const int32_t* __restrict__ verts, int64_t total, int32_t* __restrict__ cnt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[verts[e]], 1);
}
__global__ void k_fill_inc(const int32_t* __restrict__ verts, int64_t total, const int64_t* __restrict__ vptr,
                           int32_t* __restrict__ cur, int32_t* __restrict__ vlist) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int v = verts[e];
        int pos = atomicAdd(&cur[v], 1);
        vlist[vptr[v] + pos] = (int32_t)e;  // e = j*kc + slot
    }
}
__global__ void k_max_deg(const int64_t* __restrict__ vptr, int32_t nv, int32_t* out) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < nv) atomicMax(out, (int32_t)(vptr[v + 1] - vptr[v]));
}

// ----------------------------------------------------------------------------- pattern
// Warp per row: gather the incident constraints of the row's kc vertices into shared memory,
// de-duplicate and rank them (sorted ascending), diagonal last.  mode 0: count, mode 1: fill.
template <int MODE>
__global__ void k_pattern(const int32_t* __restrict__ verts, int32_t m, int kc, const int64_t* __restrict__ vptr,
                          const int32_t* __restrict__ vlist, int maxc, int32_t* __restrict__ cnt,
                          const int64_t* __restrict__ rowptr, int32_t* __restrict__ col) {
    extern __shared__ int32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t* cand = smem + warp * (2 * maxc);
    int32_t* first = cand + maxc;
    const int wpb = blockDim.x >> 5;
    for (int32_t i = blockIdx.x * wpb + warp; i < m; i += gridDim.x * wpb) {
        int64_t b0[4], len[4];
        int64_t C = 0;
        for (int k = 0; k < kc; ++k) {
            int v = verts[(int64_t)i * kc + k];
            b0[k] = vptr[v];
            len[k] = vptr[v + 1] - vptr[v];
            C += len[k];
        }
        for (int64_t p = lane; p < C; p += 32) {
            int64_t q = p;
            int k = 0;
            while (q >= len[k]) { q -= len[k]; ++k; }
            int32_t j = vlist[b0[k] + q] / kc;
            cand[p] = (j == i) ? INT_MAX : j;
        }
        __syncwarp();
        for (int64_t p = lane; p < C; p += 32) {
            int32_t v = cand[p];
            int f = (v != INT_MAX);
            for (int64_t q = 0; q < p && f; ++q) f = (cand[q] != v);
            first[p] = f;
        }
        __syncwarp();
        if (MODE == 0) {
            int c = 0;
            for (int64_t p = lane; p < C; p += 32) c += first[p];
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) cnt[i] = c + 1;
        } else {
            int64_t base = rowptr[i];
            for (int64_t p = lane; p < C; p += 32) {
                if (!first[p]) continue;
                int32_t v = cand[p];
                int r = 0;
                for (int64_t q = 0; q < C; ++q) r += (first[q] && cand[q] < v);
                col[base + r] = v;
            }
            if (lane == 0) col[rowptr[i + 1] - 1] = i;
        }
        __syncwarp();
    }
}

// ----------------------------------------------------------------------------- eval

// Polar rotation of F via the symmetric eigen-decomposition F^T F = V L V^T
// (cyclic Jacobi), sigma = sqrt(L), U = F V / sigma (completed by cross products when rank-deficient),
// R = U V^T with the smallest-sigma column of U negated when det(R) < 0.  F = 0 -> I.
__device__ void polar_rotation(const double F[9], double R[9]) {
    double S[9];
    bool zero = true;
    for (int k = 0; k < 9; ++k) zero = zero && (F[k] == 0.0);
    if (zero) {
        for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? 1.0 : 0.0;
        return;
    }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) S[r * 3 + c] = F[r] * F[c] + F[3 + r] * F[3 + c] + F[6 + r] * F[6 + c];
    double V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int sweep = 0; sweep < 16; ++sweep) {
        double off = fabs(S[1]) + fabs(S[2]) + fabs(S[5]);
        double dg = fabs(S[0]) + fabs(S[4]) + fabs(S[8]);
        if (off <= 1e-17 * dg) break;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int p = t == 2 ? 1 : 0, q = t == 0 ? 1 : 2;
            double apq = S[p * 3 + q];
            if (apq == 0.0) continue;
            // t = sgn(th) / (|th| + sqrt(th^2 + 1)) with th = u / v, c = 1 / sqrt(1 + t^2), s = t c, written
            // with w = |u| + sqrt(u^2 + v^2): t = sgn |v| / w, c = w / sqrt(w^2 + v^2), s = sgn |v| / sqrt(.) —
            // one sqrt and one rsqrt per rotation instead of two divides and two square roots (the kernel
            // is bound by the special-function unit)
            const double u = S[q * 3 + q] - S[p * 3 + p], v = 2.0 * apq;
            const double sg = (u == 0.0) ? 1.0 : ((u > 0.0) == (v > 0.0) ? 1.0 : -1.0);  // sgn(th), +1 at 0
            const double w = fabs(u) + sqrt(u * u + v * v);
            const double iq = rsqrt(w * w + v * v);
            const double c = w * iq, s = sg * fabs(v) * iq;
            // S <- J^T S J with J = rotation in (p,q)
            for (int k = 0; k < 3; ++k) {
                double skp = S[k * 3 + p], skq = S[k * 3 + q];
                S[k * 3 + p] = c * skp - s * skq;
                S[k * 3 + q] = s * skp + c * skq;
            }
            for (int k = 0; k < 3; ++k) {
                double spk = S[p * 3 + k], sqk = S[q * 3 + k];
                S[p * 3 + k] = c * spk - s * sqk;
                S[q * 3 + k] = s * spk + c * sqk;
            }
            for (int k = 0; k < 3; ++k) {
                double vkp = V[k * 3 + p], vkq = V[k * 3 + q];
                V[k * 3 + p] = c * vkp - s * vkq;
                V[k * 3 + q] = s * vkp + c * vkq;
            }
        }
    }
    double ev[3] = {S[0], S[4], S[8]};
    int o[3] = {0, 1, 2};
    if (ev[o[1]] > ev[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
    if (ev[o[2]] > ev[o[1]]) { int t = o[1]; o[1] = o[2]; o[2] = t; }
    if (ev[o[1]] > ev[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
    double Vs[9], U[9], sg[3];
    for (int k = 0; k < 3; ++k) {
        sg[k] = sqrt(fmax(ev[o[k]], 0.0));
        for (int r = 0; r < 3; ++r) Vs[r * 3 + k] = V[r * 3 + o[k]];
    }
    int rank = 0;
    for (int k = 0; k < 3; ++k) {
        double u0 = F[0] * Vs[k] + F[1] * Vs[3 + k] + F[2] * Vs[6 + k];
        double u1 = F[3] * Vs[k] + F[4] * Vs[3 + k] + F[5] * Vs[6 + k];
        double u2 = F[6] * Vs[k] + F[7] * Vs[3 + k] + F[8] * Vs[6 + k];
        const double n2 = u0 * u0 + u1 * u1 + u2 * u2;
        const double rn = n2 > 0.0 ? rsqrt(n2) : 0.0;  // one special-function op instead of sqrt + 3 divides
        const double nu = n2 * rn;
        if (nu > 1e-14 * sg[0] && rank == k) {
            U[k] = u0 * rn; U[3 + k] = u1 * rn; U[6 + k] = u2 * rn;
            rank = k + 1;
        }
    }
    if (rank < 2) {
        double a0 = U[0], a1 = U[3], a2 = U[6];
        double e0 = 0, e1 = 0, e2 = 0;
        if (fabs(a0) <= fabs(a1) && fabs(a0) <= fabs(a2)) e0 = 1; else if (fabs(a1) <= fabs(a2)) e1 = 1; else e2 = 1;
        double c0 = a1 * e2 - a2 * e1, c1 = a2 * e0 - a0 * e2, c2 = a0 * e1 - a1 * e0;
        double nn = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
        U[1] = c0 / nn; U[4] = c1 / nn; U[7] = c2 / nn;
    }
    if (rank < 3) {
        U[2] = U[3] * U[7] - U[6] * U[4];
        U[5] = U[6] * U[1] - U[0] * U[7];
        U[8] = U[0] * U[4] - U[3] * U[1];
    }
    for (int pass = 0; pass < 2; ++pass) {
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                R[r * 3 + c] = U[r * 3] * Vs[c * 3] + U[r * 3 + 1] * Vs[c * 3 + 1] + U[r * 3 + 2] * Vs[c * 3 + 2];
        double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                     R[2] * (R[3] * R[7] - R[4] * R[6]);
        if (det >= 0.0) break;
        U[2] = -U[2]; U[5] = -U[5]; U[8] = -U[8];
    }
}

// Polar rotation of F with det F > 0 by Higham's scaled Newton iteration X <- (g X + X^-T / g) / 2 (X^-T from
// the cofactor matrix, Frobenius-norm scaling g while far from convergence): for det F > 0 the orthogonal polar
// factor is the closest rotation (reading c15), reached to rounding in ~6-9 iterations of ~70 flops instead of
// the Jacobi eigen-decomposition's dozens of fp64 square roots.  Returns false (R untouched) for det F <= 0 or
// a stalled iteration: the caller falls back to polar_rotation (rank deficiency, inversion flips).
__device__ bool polar_newton(const double F[9], double R[9]) {
    double X[9];
    double nf = 0.0;
    for (int k = 0; k < 9; ++k) { X[k] = F[k]; nf += F[k] * F[k]; }
    const double det0 = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                        F[2] * (F[3] * F[7] - F[4] * F[6]);
    if (!(det0 > 1e-9 * nf * sqrt(nf))) return false;   // (near-)singular or inverted
    bool scale = true;
    for (int it = 0; it < 24; ++it) {
        double C[9];  // cofactor matrix: X^-T = C / det
        C[0] = X[4] * X[8] - X[5] * X[7]; C[1] = X[5] * X[6] - X[3] * X[8]; C[2] = X[3] * X[7] - X[4] * X[6];
        C[3] = X[2] * X[7] - X[1] * X[8]; C[4] = X[0] * X[8] - X[2] * X[6]; C[5] = X[1] * X[6] - X[0] * X[7];
        C[6] = X[1] * X[5] - X[2] * X[4]; C[7] = X[2] * X[3] - X[0] * X[5]; C[8] = X[0] * X[4] - X[1] * X[3];
        const double det = X[0] * C[0] + X[1] * C[1] + X[2] * C[2];
        if (!(det > 0.0)) return false;
        // X <- a X + c C.  Any a, c > 0 keep the polar factor of X (X = U H -> U (a H + c det H^-1)), so the
        // scaled steps take g, a, c from single-precision norms (fast sqrt / divide): only the final unscaled
        // steps, whose fixed point needs a + c det = 1 exactly, use the fp64 divide
        double a = 0.5, c;
        if (scale) {
            float nx = 0.0f, nc = 0.0f;
            for (int k = 0; k < 9; ++k) { nx += (float)X[k] * (float)X[k]; nc += (float)C[k] * (float)C[k]; }
            const float detf = (float)det;
            const float g = sqrtf(sqrtf(nc / (nx * detf * detf)));   // (||X^-1||_F / ||X||_F)^(1/2)
            a = 0.5 * (double)g;
            c = (double)(0.5f / (g * detf));
        } else {
            c = 0.5 / det;
        }
        double d2 = 0.0, n2 = 0.0;
        for (int k = 0; k < 9; ++k) {
            const double xn = a * X[k] + c * C[k];
            d2 += (xn - X[k]) * (xn - X[k]);
            n2 += xn * xn;
            X[k] = xn;
        }
        if (d2 < 1e-4 * n2) scale = false;        // close: plain Newton (quadratic) from here
        if (d2 <= 1e-30 * n2) {
            for (int k = 0; k < 9; ++k) R[k] = X[k];
            return true;
        }
    }
    return false;
}

// the vertex-major operator data of row j from its KC x 3 gradient record o (EvalHv; k_mf_refresh's arithmetic)
template <class T, int KC>
__device__ __forceinline__ void write_hv(const EvalHv<T>& e, int32_t j, const T (&o)[KC * 3], double a) {
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
        const int64_t p = e.inv[(int64_t)j * KC + k];
        e.hv[p] = o[3 * k];
        e.hv[e.npad + p] = o[3 * k + 1];
        e.hv[2 * e.npad + p] = o[3 * k + 2];
        d += (double)o[3 * k] * o[3 * k] + (double)o[3 * k + 1] * o[3 * k + 1] + (double)o[3 * k + 2] * o[3 * k + 2];
    }
    d += a;
    e.at[j] = (T)a;
    e.dinv[j] = (T)(1.0 / (double)(T)d);
}

template <class T, bool HV = false>
__global__ void k_eval_distance(int32_t m, const int32_t* __restrict__ verts, const double* __restrict__ x,
                                const double* __restrict__ L, const double* __restrict__ sqrtw,
                                const double* __restrict__ alpha, double dt2, const double* __restrict__ lambda,
                                T* __restrict__ h, T* __restrict__ b, const EvalHv<T> ehv) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    int2 ab = reinterpret_cast<const int2*>(verts)[j];
    double d0 = x[3 * ab.x] - x[3 * ab.y], d1 = x[3 * ab.x + 1] - x[3 * ab.y + 1], d2 = x[3 * ab.x + 2] - x[3 * ab.y + 2];
    double len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    double C = len - L[j];
    double il = len > 1e-12 ? 1.0 / len : 0.0;
    double u0 = d0 * il, u1 = d1 * il, u2 = d2 * il;
    double wa = sqrtw[ab.x], wb = sqrtw[ab.y];
    T* hj = h + 6 * (int64_t)j;
    const T o[6] = {(T)(wa * u0), (T)(wa * u1), (T)(wa * u2), (T)(-wb * u0), (T)(-wb * u1), (T)(-wb * u2)};
    for (int k = 0; k < 6; ++k) hj[k] = o[k];
    const double a = alpha[j] / dt2;
    if (HV) write_hv<T, 2>(ehv, j, o, a);
    b[j] = (T)(-C - a * lambda[j]);
}

// ARAP (Eq. 8, literal squared form, reading c15): C = ||F - R||_F^2, G = 2(F - R) D_m^-T,
// grad_{1..3} = columns of G, grad_0 = -sum; h_k = sqrt(w_{v_k}) grad_k.
#ifndef MGPBD_EVAL_BS
#define MGPBD_EVAL_BS 128
#endif
#ifndef MGPBD_EVAL_MINB
#define MGPBD_EVAL_MINB 8
#endif
template <class T, bool HV>
__global__ void __launch_bounds__(MGPBD_EVAL_BS, MGPBD_EVAL_MINB) k_eval_arap(int32_t m, const int32_t* __restrict__ verts, const double* __restrict__ x,
                            const double* __restrict__ Dminv, const double* __restrict__ sqrtw,
                            const double* __restrict__ alpha, double dt2, const double* __restrict__ lambda,
                            T* __restrict__ h, T* __restrict__ b, const EvalHv<T> ehv) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    int4 tv = reinterpret_cast<const int4*>(verts)[j];
    const int vv[4] = {tv.x, tv.y, tv.z, tv.w};
    double x0[3] = {x[3 * vv[0]], x[3 * vv[0] + 1], x[3 * vv[0] + 2]};
    double Ds[9];
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) Ds[r * 3 + c] = x[3 * vv[1 + c] + r] - x0[r];
    const double* Di = Dminv + 9 * (int64_t)j;
    double Dm[9];
    for (int k = 0; k < 9; ++k) Dm[k] = Di[k];
    double F[9];
    bool finite = true;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = Ds[r * 3] * Dm[c] + Ds[r * 3 + 1] * Dm[3 + c] + Ds[r * 3 + 2] * Dm[6 + c];
            F[r * 3 + c] = s;
            finite = finite && isfinite(s);
        }
    T* hj = h + 12 * (int64_t)j;
    double C = 0.0;
    const double aj = alpha[j] / dt2;
    if (!finite) {
        for (int k = 0; k < 12; ++k) hj[k] = (T)0;
        if (HV) {
            T z[12];
            for (int k = 0; k < 12; ++k) z[k] = (T)0;
            write_hv<T, 4>(ehv, j, z, aj);
        }
    } else {
        double R[9], E[9];
        if (!polar_newton(F, R)) polar_rotation(F, R);
        for (int k = 0; k < 9; ++k) { E[k] = F[k] - R[k]; C += E[k] * E[k]; }
        double g[4][3];
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r)
                g[1 + c][r] = 2.0 * (E[r * 3] * Dm[c * 3] + E[r * 3 + 1] * Dm[c * 3 + 1] + E[r * 3 + 2] * Dm[c * 3 + 2]);
        for (int r = 0; r < 3; ++r) g[0][r] = -(g[1][r] + g[2][r] + g[3][r]);
        T o[12];
        for (int k = 0; k < 4; ++k) {
            double sw = sqrtw[vv[k]];
            for (int r = 0; r < 3; ++r) o[3 * k + r] = (T)(sw * g[k][r]);
        }
        if (sizeof(T) == 4) {  // 48-byte record as three 16-byte stores (full sectors, no partial writes)
            float4* d = reinterpret_cast<float4*>(hj);
            d[0] = make_float4((float)o[0], (float)o[1], (float)o[2], (float)o[3]);
            d[1] = make_float4((float)o[4], (float)o[5], (float)o[6], (float)o[7]);
            d[2] = make_float4((float)o[8], (float)o[9], (float)o[10], (float)o[11]);
        } else {
            double2* d = reinterpret_cast<double2*>(hj);
            for (int k = 0; k < 6; ++k) d[k] = make_double2((double)o[2 * k], (double)o[2 * k + 1]);
        }
        if (HV) write_hv<T, 4>(ehv, j, o, aj);
    }
    b[j] = (T)(-C - aj * lambda[j]);
}

// ----------------------------------------------------------------------------- assembly
// ascending vertex order of a constraint's slots (compare-exchange network, static indices)
template <class T, int KC>
__device__ __forceinline__ void sort_slots(int (&v)[KC], T (&hh)[KC][3]) {
    auto cx = [&](int a, int b) {
        const bool sw = v[b] < v[a];
        const int ta = v[a], tb = v[b];
        v[a] = sw ? tb : ta;
        v[b] = sw ? ta : tb;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const T xa = hh[a][r], xb = hh[b][r];
            hh[a][r] = sw ? xb : xa;
            hh[b][r] = sw ? xa : xb;
        }
    };
    if constexpr (KC == 4) { cx(0, 1); cx(2, 3); cx(0, 2); cx(1, 3); cx(1, 2); }
    else cx(0, 1);
}

// Sub-warp (VL lanes) per row.  A_ij = sum over shared vertices (ascending vertex id) of
// h_{i,v} . h_{j,v}; A_ii = sum_k |h_{i,k}|^2 + alpha_i/dt^2 (reading c14).
template <class T, int KC, int VL>
__global__ void __launch_bounds__(256) k_assemble(int32_t row0, int32_t m, const int32_t* __restrict__ verts, const T* __restrict__ h,
                                                  const double* __restrict__ alpha, double dt2,
                                                  const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                                  T* __restrict__ val, T* __restrict__ dinv) {
    const int sub = threadIdx.x % VL;
    const int64_t gsub = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / VL;
    const int64_t nsub = (int64_t)gridDim.x * blockDim.x / VL;
    using IV = typename std::conditional<KC == 4, int4, int2>::type;
    for (int64_t i = row0 + gsub; i < m; i += nsub) {  // rows [row0, m)
        int vi[KC];
        T hi[KC][3];
        {
            const IV v4 = reinterpret_cast<const IV*>(verts)[i];
            load_iv(v4, vi);
            load_record<T, KC>(h + i * KC * 3, hi);
        }
        // diagonal (slot order), before the rows' vertices are sorted
        double d = 0.0;
#pragma unroll
        for (int k = 0; k < KC; ++k)
            d += (double)hi[k][0] * hi[k][0] + (double)hi[k][1] * hi[k][1] + (double)hi[k][2] * hi[k][2];
        // ascending vertex order of row i's vertices: compare-exchange network with static indices
        // (keeps vi/hi in registers)
        sort_slots<T, KC>(vi, hi);
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1] - 1;
        for (int64_t e = e0 + sub; e < e1; e += VL) {
            const int32_t j = col[e];
            int vj[KC];
            T hj[KC][3];
            load_iv(reinterpret_cast<const IV*>(verts)[j], vj);
            load_record<T, KC>(h + (int64_t)j * KC * 3, hj);  // whole record, 16-byte vectors
            double s = 0.0;
#pragma unroll
            for (int t = 0; t < KC; ++t) {
#pragma unroll
                for (int q = 0; q < KC; ++q) {
                    if (vj[q] == vi[t])
                        s += (double)hi[t][0] * hj[q][0] + (double)hi[t][1] * hj[q][1] + (double)hi[t][2] * hj[q][2];
                }
            }
            val[e] = (T)s;
        }
        if (sub == 0) {
            d += alpha[i] / dt2;
            val[e1] = (T)d;
            dinv[i] = (T)(1.0 / (double)(T)d);
        }
    }
}

// ----------------------------------------------------------------------------- vertex kernels
__global__ void k_predict(int32_t n, double* __restrict__ x, double* __restrict__ v, double* __restrict__ x_old,
                          const double* __restrict__ w, double dt, double gx, double gy, double gz) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double g[3] = {gx, gy, gz};
    bool free_ = w[i] > 0.0;
    for (int r = 0; r < 3; ++r) {
        double xi = x[3 * i + r], vi = v[3 * i + r];
        x_old[3 * i + r] = xi;
        if (free_) vi += dt * g[r];
        v[3 * i + r] = vi;
        x[3 * i + r] = xi + dt * vi;
    }
}

// dx_v = sqrt(w_v) sum_{(j,k) incident, ascending j} h_{j,k} dl_j (Eq. 5); x += omega dx (Alg. 1 l.11)
template <class T>
__global__ void k_update(int32_t n, int kc, const int64_t* __restrict__ vptr, const int32_t* __restrict__ vlist,
                         const T* __restrict__ h, const double* __restrict__ sqrtw, const T* __restrict__ dl,
                         const double* __restrict__ omega_p, double* __restrict__ x) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    double s0 = 0, s1 = 0, s2 = 0;
    for (int64_t e = vptr[v]; e < vptr[v + 1]; ++e) {
        int32_t code = vlist[e];
        int32_t j = code / kc;
        const T* hh = h + (int64_t)code * 3;
        double d = (double)dl[j];
        s0 += (double)hh[0] * d; s1 += (double)hh[1] * d; s2 += (double)hh[2] * d;
    }
    const double sw = sqrtw[v], omega = *omega_p;
    x[3 * v] += omega * (sw * s0);
    x[3 * v + 1] += omega * (sw * s1);
    x[3 * v + 2] += omega * (sw * s2);
}

template <class T>
__global__ void k_lambda_add(int32_t m, double* __restrict__ lambda, const T* __restrict__ dl) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < m) lambda[j] += (double)dl[j];
}
__global__ void k_velocity(int32_t n3, const double* __restrict__ x, const double* __restrict__ x_old,
                           double* __restrict__ v, double dt) {
    int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n3) v[k] = (x[k] - x_old[k]) / dt;
}
__global__ void k_sqrt(int32_t n, const double* __restrict__ w, double* __restrict__ o) {
    int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) o[k] = sqrt(w[k]);
}

}  // namespace

void rest_distance(const int32_t* verts, const double* X, int32_t m, double* L, cudaStream_t s) {
    if (!m) return;
    k_rest_distance<<<grid1d(m), 256, 0, s>>>(verts, X, m, L);
    MG_LAUNCH_CHECK();
}
void rest_arap(const int32_t* verts, const double* X, int32_t m, double* Dminv, double* vol, int32_t* bad,
               cudaStream_t s) {
    if (!m) return;
    k_rest_arap<<<grid1d(m), 256, 0, s>>>(verts, X, m, Dminv, vol, bad);
    MG_LAUNCH_CHECK();
}

void build_incidence(const int32_t* verts, int32_t m, int kc, int32_t nv, DBuf<int64_t>& vptr,
                     DBuf<int32_t>& vlist, cudaStream_t s) {
    int64_t total = (int64_t)m * kc;
    DBuf<int32_t> cnt;
    cnt.resize(nv);
    vptr.resize(nv + 1);
    vlist.resize(total);
    MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (nv ? nv : 1), s));
    int g = (int)std::min<int64_t>(grid1d(total), 148 * 32);
    if (total) { k_count_inc<<<g, 256, 0, s>>>(verts, total, cnt.p); MG_LAUNCH_CHECK(); }
    scan_exclusive<int32_t>(cnt.p, vptr.p, nv, s);
    MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (nv ? nv : 1), s));
    if (total) { k_fill_inc<<<g, 256, 0, s>>>(verts, total, vptr.p, cnt.p, vlist.p); MG_LAUNCH_CHECK(); }
    sort_segments_i32(vptr.p, vlist.p, nv, s);
    MG_CK(cudaStreamSynchronize(s));
}

void build_pattern(const int32_t* verts, int32_t m, int kc, int32_t nv, const int64_t* vptr, const int32_t* vlist,
                   DBuf<int64_t>& rowptr, DBuf<int32_t>& col, cudaStream_t s) {
    DBuf<int32_t> md;
    md.resize(1);
    MG_CK(cudaMemsetAsync(md.p, 0, sizeof(int32_t), s));
    if (nv) { k_max_deg<<<grid1d(nv), 256, 0, s>>>(vptr, nv, md.p); MG_LAUNCH_CHECK(); }
    int32_t maxdeg = read_scalar(md.p, s);
    int maxc = std::max(1, maxdeg * kc);
    size_t per_warp = (size_t)maxc * 2 * sizeof(int32_t);
    int wpb = 8;
    while (wpb > 1 && per_warp * wpb > 96 * 1024) wpb >>= 1;
    if (per_warp * wpb > 200 * 1024) throw Error(-1, "vertex degree too large for the pattern kernel");
    size_t smem = per_warp * wpb;
    if (smem > 48 * 1024) {
        ensure_dyn_smem((const void*)k_pattern<0>, smem);
        ensure_dyn_smem((const void*)k_pattern<1>, smem);
    }
    DBuf<int32_t> cnt;
    cnt.resize(m);
    rowptr.resize(m + 1);
    int grid = (int)std::min<int64_t>(ceil_div(m, wpb), 148 * 64);
    if (m) { k_pattern<0><<<grid, 32 * wpb, smem, s>>>(verts, m, kc, vptr, vlist, maxc, cnt.p, nullptr, nullptr); MG_LAUNCH_CHECK(); }
    scan_exclusive<int32_t>(cnt.p, rowptr.p, m, s);
    int64_t nnz = read_scalar(rowptr.p + m, s);
    col.resize(nnz);
    if (m) { k_pattern<1><<<grid, 32 * wpb, smem, s>>>(verts, m, kc, vptr, vlist, maxc, nullptr, rowptr.p, col.p); MG_LAUNCH_CHECK(); }
    MG_CK(cudaStreamSynchronize(s));
}

template <class T>
void eval_constraints(int kind, int32_t m, const int32_t* verts, const double* x, const double* rest,
                      const double* sqrtw, const double* alpha, double dt, const double* lambda, T* h, T* b,
                      cudaStream_t s, const EvalHv<T>* hvout) {
    if (!m) return;
    double dt2 = dt * dt;
    const EvalHv<T> e = hvout ? *hvout : EvalHv<T>();
    if (kind == 2) {
        if (hvout) k_eval_distance<T, true><<<grid1d(m), 256, 0, s>>>(m, verts, x, rest, sqrtw, alpha, dt2, lambda, h, b, e);
        else k_eval_distance<T, false><<<grid1d(m), 256, 0, s>>>(m, verts, x, rest, sqrtw, alpha, dt2, lambda, h, b, e);
    } else {
        if (hvout)
            k_eval_arap<T, true><<<grid1d(m, MGPBD_EVAL_BS), MGPBD_EVAL_BS, 0, s>>>(m, verts, x, rest, sqrtw, alpha, dt2, lambda, h, b, e);
        else
            k_eval_arap<T, false><<<grid1d(m, MGPBD_EVAL_BS), MGPBD_EVAL_BS, 0, s>>>(m, verts, x, rest, sqrtw, alpha, dt2, lambda, h, b, e);
    }
    MG_LAUNCH_CHECK();
}

template <class T>
void assemble(int kind, int32_t m, const int32_t* verts, const T* h, const double* alpha, double dt,
              const int64_t* rowptr, const int32_t* col, int vl, T* val, T* dinv, cudaStream_t s, int32_t row0,
              int32_t row1) {
    if (row1 < 0) row1 = m;
    if (row1 <= row0) return;
    double dt2 = dt * dt;
    int64_t threads = (int64_t)(row1 - row0) * vl;
    int grid = (int)std::min<int64_t>((threads + 255) / 256, 148 * 16);
#define MG_ASM(KC, VL) k_assemble<T, KC, VL><<<grid, 256, 0, s>>>(row0, row1, verts, h, alpha, dt2, rowptr, col, val, dinv)
    if (kind == 2) {
        if (vl <= 4) MG_ASM(2, 4); else if (vl <= 8) MG_ASM(2, 8); else MG_ASM(2, 16);
    } else {
        if (vl <= 8) MG_ASM(4, 8); else if (vl <= 16) MG_ASM(4, 16); else MG_ASM(4, 32);
    }
#undef MG_ASM
    MG_LAUNCH_CHECK();
}

void predict(int32_t n, double* x, double* v, double* x_old, const double* w, double dt, double gx, double gy,
             double gz, cudaStream_t s) {
    if (!n) return;
    k_predict<<<grid1d(n), 256, 0, s>>>(n, x, v, x_old, w, dt, gx, gy, gz);
    MG_LAUNCH_CHECK();
}
template <class T>
void update_positions(int32_t n, int kc, const int64_t* vptr, const int32_t* vlist, const T* h, const double* sqrtw,
                      const T* dl, const double* omega, double* x, cudaStream_t s) {
    if (!n) return;
    k_update<T><<<grid1d(n, 128), 128, 0, s>>>(n, kc, vptr, vlist, h, sqrtw, dl, omega, x);
    MG_LAUNCH_CHECK();
}
template <class T>
void lambda_add(int32_t m, double* lambda, const T* dl, cudaStream_t s) {
    if (!m) return;
    k_lambda_add<T><<<grid1d(m), 256, 0, s>>>(m, lambda, dl);
    MG_LAUNCH_CHECK();
}
// Backtracking relaxation (reading c21): omega /= 2 (floored at omega_min) when the
// squared residual norm of outer iteration ite exceeds that of ite - 1.  One thread; graph-safe.
__global__ void k_backtrack(const double* __restrict__ bn2, int ite, double* __restrict__ omega, double omega_min) {
    if (ite > 0 && bn2[ite] > bn2[ite - 1]) *omega = fmax(0.5 * *omega, omega_min);
}
void backtrack_omega(const double* bn2, int ite, double* omega, double omega_min, cudaStream_t s) {
    k_backtrack<<<1, 1, 0, s>>>(bn2, ite, omega, omega_min);
    MG_LAUNCH_CHECK();
}

void velocity(int32_t n, const double* x, const double* x_old, double* v, double dt, cudaStream_t s) {
    if (!n) return;
    k_velocity<<<grid1d(3 * (int64_t)n), 256, 0, s>>>(3 * n, x, x_old, v, dt);
    MG_LAUNCH_CHECK();
}
void sqrt_vec(int32_t n, const double* w, double* out, cudaStream_t s) {
    if (!n) return;
    k_sqrt<<<grid1d(n), 256, 0, s>>>(n, w, out);
    MG_LAUNCH_CHECK();
}

#define MG_INST(T)                                                                                          \
    template void eval_constraints<T>(int, int32_t, const int32_t*, const double*, const double*, const double*, \
                                      const double*, double, const double*, T*, T*, cudaStream_t,            \
                                      const EvalHv<T>*);                                                     \
    template void assemble<T>(int, int32_t, const int32_t*, const T*, const double*, double, const int64_t*,  \
                              const int32_t*, int, T*, T*, cudaStream_t, int32_t, int32_t);                  \
    template void update_positions<T>(int32_t, int, const int64_t*, const int32_t*, const T*, const double*,  \
                                      const T*, const double*, double*, cudaStream_t);                       \
    template void lambda_add<T>(int32_t, double*, const T*, cudaStream_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mgpbd
