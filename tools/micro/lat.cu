// Microbenchmark: dependent-chain latency (cycles) of fp64 ops, shuffles and barriers on one warp / CTA.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
    double a = seed + threadIdx.x * 1e-9, b = 1.0 + seed;
    long long t0, t1;
    const int N = 256;
    // fp64 fma chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = fma(a, b, 1e-7);
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
    // fp64 divide chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = 1.0 / (a + 1.5);
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / N;
    // __drcp_rn chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = __drcp_rn(a + 1.5);
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / N;
    // shfl double chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = __shfl_sync(0xffffffffu, a, i & 31) + 1e-9;
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / N;
    // shfl float chain
    float f = (float)a;
    t0 = clock64();
    for (int i = 0; i < N; ++i) f = __shfl_sync(0xffffffffu, f, i & 31) + 1e-9f;
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / N;
    // syncthreads + smem round trip chain
    __shared__ double s[1024];
    t0 = clock64();
    for (int i = 0; i < N; ++i) { s[threadIdx.x] = a; __syncthreads(); a = s[(threadIdx.x + 1) % blockDim.x] + 1e-9; __syncthreads(); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / N;
    // independent shfl throughput: 32 independent shuffles
    double v[32];
    for (int j = 0; j < 32; ++j) v[j] = a + j;
    t0 = clock64();
    for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __shfl_sync(0xffffffffu, v[j], (i + j) & 31);
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / 8;
    for (int j = 0; j < 32; ++j) a += v[j];
    out[threadIdx.x] = a + f;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64 * 8);
    for (int bs : {32, 256}) {
        k<<<1, bs>>>(o, c, 0.5);
        long long h[8]; cudaMemcpy(h, c, 7 * 8, cudaMemcpyDeviceToHost);
        printf("block %d: fma %lld, div %lld, drcp %lld, shfl64 %lld, shfl32 %lld, sync+smem %lld, 32 indep shfl64 %lld cycles\n",
               bs, h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
    }
}
