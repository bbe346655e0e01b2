// Microbenchmark: the cooperative blocked Gauss-Jordan inverse (csrc/solve.cu k_gj_coop) on a random SPD
// n x n matrix, with per-phase device timestamps of CTA 0 (globaltimer), to see where a panel's time goes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/gj tools/micro/gj.cu && tools/micro/gj 357
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int GJT = 256;
template <bool STAMP>
__global__ void __launch_bounds__(GJT) k_gj(int32_t n, const double* __restrict__ A, double* W0, double* W1,
                                           unsigned long long* st) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double Ps[32][33];
    __shared__ double Ks[32][33];
    __shared__ double Cs[32][33];
    __shared__ double Rs[32][33];
    const int npan = (n + 31) / 32;
    double* cur = (npan % 2 == 0) ? W0 : W1;
    double* nxt = (npan % 2 == 0) ? W1 : W0;
    const bool rec = STAMP && blockIdx.x == 0 && threadIdx.x == 0;
    int si = 0;
    if (rec) st[si++] = gtime();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)n * n; q += (int64_t)gridDim.x * blockDim.x)
        cur[q] = A[q];
    grid.sync();
    if (rec) st[si++] = gtime();
    for (int pnl = 0; pnl < npan; ++pnl) {
        const int32_t k0 = pnl * 32, bs = min(32, n - k0);
        for (int q = threadIdx.x; q < 32 * 32; q += GJT) {
            const int i = q >> 5, j = q & 31;
            Ps[i][j] = (i < bs && j < bs) ? cur[(int64_t)(k0 + i) * n + k0 + j] : (i == j ? 1.0 : 0.0);
        }
        __syncthreads();
        if (rec) st[si++] = gtime();
        for (int k = 0; k < 32; ++k) {
            double pv = Ps[k][k];
            const double ip = 1.0 / pv;
            double nv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = threadIdx.x + u * GJT, i = q >> 5, j = q & 31;
                const double sij = Ps[i][j], sik = Ps[i][k], skj = Ps[k][j];
                nv[u] = i == k ? (j == k ? ip : skj * ip) : (j == k ? -sik * ip : sij - sik * skj * ip);
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = threadIdx.x + u * GJT;
                Ps[q >> 5][q & 31] = nv[u];
            }
            __syncthreads();
        }
        if (rec) st[si++] = gtime();
        const int nt = npan * npan;
        for (int tile = blockIdx.x; tile < nt; tile += gridDim.x) {
            const int I = tile / npan, J = tile % npan;
            const int32_t i0 = I * 32, j0 = J * 32;
            const bool iK = I == pnl, jK = J == pnl;
            for (int q = threadIdx.x; q < 32 * 32; q += GJT) {
                const int r = q >> 5, c = q & 31;
                if (!jK) Ks[r][c] = (r < bs && j0 + c < n) ? cur[(int64_t)(k0 + r) * n + j0 + c] : 0.0;
                if (!iK) Cs[r][c] = (i0 + r < n && c < bs) ? cur[(int64_t)(i0 + r) * n + k0 + c] : 0.0;
            }
            __syncthreads();
            if (rec && tile == (int)blockIdx.x) st[si] = gtime();
            if (!jK) {
                for (int q = threadIdx.x; q < 32 * 32; q += GJT) {
                    const int t = q >> 5, c = q & 31;
                    double acc = 0.0;
#pragma unroll 8
                    for (int u = 0; u < 32; ++u) acc += Ps[t][u] * Ks[u][c];
                    Rs[t][c] = acc;
                }
            }
            __syncthreads();
            for (int q = threadIdx.x; q < 32 * 32; q += GJT) {
                const int r = q >> 5, c = q & 31;
                const int32_t i = i0 + r, j = j0 + c;
                if (i >= n || j >= n) continue;
                double v;
                if (iK && jK) v = Ps[r][c];
                else if (iK) v = Rs[r][c];
                else if (jK) {
                    double acc = 0.0;
#pragma unroll 8
                    for (int t = 0; t < 32; ++t) acc += Cs[r][t] * Ps[t][c];
                    v = -acc;
                } else {
                    double acc = 0.0;
#pragma unroll 8
                    for (int t = 0; t < 32; ++t) acc += Cs[r][t] * Rs[t][c];
                    v = cur[(int64_t)i * n + j] - acc;
                }
                nxt[(int64_t)i * n + j] = v;
            }
            __syncthreads();
        }
        if (rec) { ++si; st[si++] = gtime(); }
        grid.sync();
        if (rec) st[si++] = gtime();
        double* t = cur; cur = nxt; nxt = t;
    }
    if (rec) st[63] = si;
}


// v2: pivot block inverted by warp 0 with register-resident columns (fully unrolled: static register
// indices), tiles updated with 4 independent accumulators per thread (rows ty, ty+8, ty+16, ty+24).
template <bool STAMP>
__global__ void __launch_bounds__(GJT) k_gj2(int32_t n, const double* __restrict__ A, double* W0, double* W1,
                                            unsigned long long* st) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double Ps[32][33];
    __shared__ double Ks[32][33];
    __shared__ double Cs[32][33];
    __shared__ double Rs[32][33];
    const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int npan = (n + 31) / 32;
    double* cur = (npan % 2 == 0) ? W0 : W1;
    double* nxt = (npan % 2 == 0) ? W1 : W0;
    const bool rec = STAMP && blockIdx.x == 0 && threadIdx.x == 0;
    int si = 0;
    if (rec) st[si++] = gtime();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)n * n; q += (int64_t)gridDim.x * blockDim.x)
        cur[q] = A[q];
    grid.sync();
    if (rec) st[si++] = gtime();
    for (int pnl = 0; pnl < npan; ++pnl) {
        const int32_t k0 = pnl * 32, bs = min(32, n - k0);
        if (ty == 0) {
            double c[32];  // column `lane` of the pivot block
#pragma unroll
            for (int i = 0; i < 32; ++i)
                c[i] = (i < bs && lane < bs) ? cur[(int64_t)(k0 + i) * n + k0 + lane] : (i == lane ? 1.0 : 0.0);
            if (rec) st[si++] = gtime();
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const double pk = __shfl_sync(0xffffffffu, c[k], k);
                const double ip = 1.0 / pk;
                const double rkj = c[k] * ip;        // new pivot row entry (j != k)
                const bool jk = lane == k;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i == k) continue;
                    const double aik = __shfl_sync(0xffffffffu, c[i], k);
                    c[i] = jk ? -aik * ip : fma(-aik, rkj, c[i]);
                }
                c[k] = jk ? ip : rkj;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) Ps[i][lane] = c[i];
        }
        __syncthreads();
        if (rec) st[si++] = gtime();
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
            if (rec && tile == (int)blockIdx.x) st[si] = gtime();
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
        if (rec) { ++si; st[si++] = gtime(); }
        grid.sync();
        if (rec) st[si++] = gtime();
        double* t = cur; cur = nxt; nxt = t;
    }
    if (rec) st[63] = si;
}

// v4: v2's tiles; the pivot block inverted by the whole CTA with ping-pong buffers (one barrier per step)
// (was v2: pivot block inverted by warp 0 with register-resident columns (fully unrolled: static register
// indices), tiles updated with 4 independent accumulators per thread (rows ty, ty+8, ty+16, ty+24).
template <bool STAMP>
__global__ void __launch_bounds__(GJT) k_gj4(int32_t n, const double* __restrict__ A, double* W0, double* W1,
                                            unsigned long long* st) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double Ps[32][33];
    __shared__ double Qs[32][33];
    __shared__ double Ks[32][33];
    __shared__ double Cs[32][33];
    __shared__ double Rs[32][33];
    const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int npan = (n + 31) / 32;
    double* cur = (npan % 2 == 0) ? W0 : W1;
    double* nxt = (npan % 2 == 0) ? W1 : W0;
    const bool rec = STAMP && blockIdx.x == 0 && threadIdx.x == 0;
    int si = 0;
    if (rec) st[si++] = gtime();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)n * n; q += (int64_t)gridDim.x * blockDim.x)
        cur[q] = A[q];
    grid.sync();
    if (rec) st[si++] = gtime();
    for (int pnl = 0; pnl < npan; ++pnl) {
        const int32_t k0 = pnl * 32, bs = min(32, n - k0);
        for (int u = 0; u < 4; ++u) {
            const int i = ty + 8 * u;
            Ps[i][lane] = (i < bs && lane < bs) ? cur[(int64_t)(k0 + i) * n + k0 + lane] : (i == lane ? 1.0 : 0.0);
        }
        __syncthreads();
        if (rec) st[si++] = gtime();
#pragma unroll 2
        for (int k = 0; k < 32; ++k) {
            double (*A_)[33] = (k & 1) ? Qs : Ps;
            double (*B_)[33] = (k & 1) ? Ps : Qs;
            const double ip = 1.0 / A_[k][k];
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
        }
        __syncthreads();
        if (rec) st[si++] = gtime();
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
            if (rec && tile == (int)blockIdx.x) st[si] = gtime();
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
        if (rec) { ++si; st[si++] = gtime(); }
        grid.sync();
        if (rec) st[si++] = gtime();
        double* t = cur; cur = nxt; nxt = t;
    }
    if (rec) st[63] = si;
}

// v3: as v2, with a fast fp64 reciprocal (fp32 seed + 2 Newton steps) and the products formed before it;
// v2: pivot block inverted by warp 0 with register-resident columns (fully unrolled: static register
// indices), tiles updated with 4 independent accumulators per thread (rows ty, ty+8, ty+16, ty+24).
template <bool STAMP>
__global__ void __launch_bounds__(GJT) k_gj3(int32_t n, const double* __restrict__ A, double* W0, double* W1,
                                            unsigned long long* st) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double Ps[32][33];
    __shared__ double Ks[32][33];
    __shared__ double Cs[32][33];
    __shared__ double Rs[32][33];
    const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int npan = (n + 31) / 32;
    double* cur = (npan % 2 == 0) ? W0 : W1;
    double* nxt = (npan % 2 == 0) ? W1 : W0;
    const bool rec = STAMP && blockIdx.x == 0 && threadIdx.x == 0;
    int si = 0;
    if (rec) st[si++] = gtime();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (int64_t)n * n; q += (int64_t)gridDim.x * blockDim.x)
        cur[q] = A[q];
    grid.sync();
    if (rec) st[si++] = gtime();
    for (int pnl = 0; pnl < npan; ++pnl) {
        const int32_t k0 = pnl * 32, bs = min(32, n - k0);
        if (ty == 0) {
            double c[32];  // column `lane` of the pivot block
#pragma unroll
            for (int i = 0; i < 32; ++i)
                c[i] = (i < bs && lane < bs) ? cur[(int64_t)(k0 + i) * n + k0 + lane] : (i == lane ? 1.0 : 0.0);
            if (rec) st[si++] = gtime();
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const double pk = __shfl_sync(0xffffffffu, c[k], k);
                double ip = (double)__frcp_rn((float)pk);
                double e = fma(-pk, ip, 1.0);
                ip = fma(ip, e, ip);
                e = fma(-pk, ip, 1.0);
                ip = fma(ip, e, ip);
                const bool jk = lane == k;
                const double ckj = jk ? -1.0 : c[k];  // lane k: new column k = -a_ik / p
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i == k) continue;
                    const double aik = __shfl_sync(0xffffffffu, c[i], k);
                    c[i] = fma(-(aik * ckj), ip, jk ? 0.0 : c[i]);
                }
                c[k] = jk ? ip : c[k] * ip;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) Ps[i][lane] = c[i];
        }
        __syncthreads();
        if (rec) st[si++] = gtime();
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
            if (rec && tile == (int)blockIdx.x) st[si] = gtime();
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
        if (rec) { ++si; st[si++] = gtime(); }
        grid.sync();
        if (rec) st[si++] = gtime();
        double* t = cur; cur = nxt; nxt = t;
    }
    if (rec) st[63] = si;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 357;
    std::vector<double> A((size_t)n * n);
    srand(1);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double v = (i == j) ? n : (rand() / (double)RAND_MAX - 0.5);
            A[(size_t)i * n + j] = A[(size_t)j * n + i] = v;
        }
    double *dA, *W0, *W1; unsigned long long* st;
    cudaMalloc(&dA, 8 * A.size()); cudaMalloc(&W0, 8 * A.size()); cudaMalloc(&W1, 8 * A.size());
    cudaMalloc(&st, 8 * 2048);
    cudaMemcpy(dA, A.data(), 8 * A.size(), cudaMemcpyHostToDevice);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gj<false>, GJT, 0);
    const int npan = (n + 31) / 32;
    int G = std::min(148 * std::min(occ, 2), npan * npan);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int ver = argc > 2 ? atoi(argv[2]) : 1;
    for (int stamp = 0; stamp < 2; ++stamp) {
        void* args[] = {(void*)&n, &dA, &W0, &W1, &st};
        auto fn = ver == 4 ? (stamp ? (void*)k_gj4<true> : (void*)k_gj4<false>) : ver == 3 ? (stamp ? (void*)k_gj3<true> : (void*)k_gj3<false>) : ver == 2 ? (stamp ? (void*)k_gj2<true> : (void*)k_gj2<false>)
                           : (stamp ? (void*)k_gj<true> : (void*)k_gj<false>);
        for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel(fn, G, GJT, args, 0, 0);
        cudaEventRecord(e0);
        const int R = 20;
        for (int w = 0; w < R; ++w) cudaLaunchCooperativeKernel(fn, G, GJT, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("v%d n=%d grid=%d stamp=%d: %.1f us per inverse (%s)\n", ver, n, G, stamp, 1000 * ms / R,
               cudaGetErrorString(cudaGetLastError()));
    }
    std::vector<unsigned long long> h(2048);
    cudaMemcpy(h.data(), st, 8 * 64, cudaMemcpyDeviceToHost);
    int ns = (int)h[63];
    printf("load+sync %.2f us\n", (h[1] - h[0]) * 1e-3);
    double piv = 0, ld = 0, comp = 0, sy = 0;
    for (int p = 0; p < npan; ++p) {
        unsigned long long* s = &h[2 + 5 * p];
        piv += (s[1] - s[0]) * 1e-3; ld += (s[2] - s[1]) * 1e-3; comp += (s[3] - s[2]) * 1e-3; sy += (s[4] - s[3]) * 1e-3;
        if (p < 3) printf("panel %d: Ps load->piv %.2f, piv %.2f, tile loads %.2f, tile compute %.2f, grid.sync %.2f us\n", p,
                          0.0, (s[1] - s[0]) * 1e-3, (s[2] - s[1]) * 1e-3, (s[3] - s[2]) * 1e-3, (s[4] - s[3]) * 1e-3);
    }
    printf("stamps %d; totals: pivot %.1f, tile loads %.1f, compute %.1f, sync %.1f us\n", ns, piv, ld, comp, sy);
    // check: W * A = I
    std::vector<double> Wh(A.size());
    cudaMemcpy(Wh.data(), W0, 8 * A.size(), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0; for (int k = 0; k < n; ++k) s += Wh[(size_t)i * n + k] * A[(size_t)k * n + j];
            err = fmax(err, fabs(s - (i == j)));
        }
    printf("max |WA - I| = %.3e\n", err);
}
