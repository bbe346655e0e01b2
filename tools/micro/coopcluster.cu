// Microbenchmark: can a cooperative launch carry cluster dimensions on this GPU, and what do grid.sync and
// cluster.sync cost inside it?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 coopcluster.cu -o coopcluster
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k(int iters, int mode, int* sink) {
    cg::grid_group g = cg::this_grid();
    cg::cluster_group c = cg::this_cluster();
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += i;
        if (mode == 0) g.sync();
        else c.sync();
    }
    if (acc == -1) *sink = acc;
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        int ncl = 0;
        cfg.gridDim = dim3(cs);
        cudaError_t e0 = cudaOccupancyMaxActiveClusters(&ncl, (const void*)k, &cfg);
        cfg.gridDim = dim3(ncl * cs);
        for (int mode = 0; mode < 2; ++mode) {
            int iters = 1000;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, iters, mode, sink);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&cfg, k, iters, mode, sink);
            cudaEventRecord(b);
            cudaError_t e2 = cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("cluster %2d: %3d clusters (%3d CTAs, occ %s) %s: launch %s / %s, %.3f us per sync\n", cs, ncl,
                   ncl * cs, cudaGetErrorString(e0), mode ? "cluster.sync" : "grid.sync  ", cudaGetErrorString(e1),
                   cudaGetErrorString(e2), ms * 1e3 / iters);
            cudaGetLastError();
        }
    }
    return 0;
}
