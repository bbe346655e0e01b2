// Microbenchmark: cost of a grid-wide barrier on this GPU (cooperative groups vs a hand-rolled one).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda/atomic>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
    cg::grid_group g = cg::this_grid();
    int acc = 0;
    for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
    if (acc == -1) *sink = acc;
}

__device__ __forceinline__ void bar(unsigned* count, unsigned* gen, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> c(*count), gg(*gen);
        unsigned g0 = gg.load(cuda::memory_order_relaxed);
        if (c.fetch_add(1, cuda::memory_order_acq_rel) == nb - 1) {
            c.store(0, cuda::memory_order_relaxed);
            gg.store(g0 + 1, cuda::memory_order_release);
        } else {
            while (gg.load(cuda::memory_order_acquire) == g0) { }
        }
    }
    __syncthreads();
}
__global__ void k_own(int iters, unsigned* count, unsigned* gen, int* sink) {
    int acc = 0;
    for (int i = 0; i < iters; ++i) { acc += i; bar(count, gen, gridDim.x); }
    if (acc == -1) *sink = acc;
}

int main() {
    int* sink; unsigned* cnt; cudaMalloc(&sink, 4); cudaMalloc(&cnt, 8); cudaMemset(cnt, 0, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int cfgs[][2] = {{148, 128}, {148, 512}, {296, 512}, {148, 1024}, {74, 512}, {32, 512}};
    for (auto& c : cfgs) {
        int iters = 1000;
        void* args[] = {&iters, &sink};
        cudaLaunchCooperativeKernel((void*)k_cg, c[0], c[1], args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, c[0], c[1], args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned* gen = cnt + 1;
        void* args2[] = {&iters, &cnt, &gen, &sink};
        cudaLaunchCooperativeKernel((void*)k_own, c[0], c[1], args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_own, c[0], c[1], args2, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("grid %4d x %4d: cg::sync %.2f us, own barrier %.2f us  (%s)\n", c[0], c[1], ms * 1e3 / iters, ms2 * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
