// Deterministic scans, reductions and small helper kernels.
#include "util.cuh"

#include <map>
#include <mutex>
#include <unordered_map>

namespace mgpbd {

thread_local int64_t g_kernel_launches = 0;
thread_local cudaStream_t g_alloc_stream = nullptr;

namespace {
constexpr int SB = 1024;      // threads per scan block
constexpr int SI = 4;         // items per thread
constexpr int SCHUNK = SB * SI;

template <class TI>
__global__ void k_scan_blocksum(const TI* in, int64_t n, int64_t* bsum) {
    __shared__ int64_t sh[SB / 32];
    int64_t base = (int64_t)blockIdx.x * SCHUNK;
    int64_t v = 0;
    for (int k = 0; k < SI; ++k) {
        int64_t i = base + (int64_t)k * SB + threadIdx.x;
        if (i < n) v += (int64_t)in[i];
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t w = threadIdx.x < SB / 32 ? sh[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) bsum[blockIdx.x] = w;
    }
}

// single block exclusive scan of bsum in place (nb arbitrary), writes total to *tot
__global__ void k_scan_bsums(int64_t* bsum, int64_t nb, int64_t* tot) {
    __shared__ int64_t sh[SB];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nb; b0 += SB) {
        int64_t i = b0 + threadIdx.x;
        int64_t v = i < nb ? bsum[i] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < SB; o <<= 1) {
            int64_t t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        int64_t incl = sh[threadIdx.x];
        if (i < nb) bsum[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == SB - 1) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *tot = carry;
}

template <class TI>
__global__ void k_scan_final(const TI* in, int64_t n, const int64_t* bsum, int64_t* out) {
    __shared__ int64_t sh[SB];
    int64_t base = (int64_t)blockIdx.x * SCHUNK + (int64_t)threadIdx.x * SI;
    int64_t loc[SI];
    int64_t s = 0;
    for (int k = 0; k < SI; ++k) {
        int64_t i = base + k;
        loc[k] = s;
        s += (i < n) ? (int64_t)in[i] : 0;
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < SB; o <<= 1) {
        int64_t t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
        __syncthreads();
        sh[threadIdx.x] += t;
        __syncthreads();
    }
    int64_t off = bsum[blockIdx.x] + sh[threadIdx.x] - s;
    for (int k = 0; k < SI; ++k) {
        int64_t i = base + k;
        if (i < n) out[i] = off + loc[k];
    }
}
}  // namespace

template <class TI>
void scan_exclusive(const TI* in, int64_t* out, int64_t n, cudaStream_t s) {
    int64_t nb = (n + SCHUNK - 1) / SCHUNK;
    if (nb == 0) { MG_CK(cudaMemsetAsync(out, 0, sizeof(int64_t), s)); return; }
    int64_t* bsum;
    MG_CK(cudaMallocAsync(&bsum, sizeof(int64_t) * nb, s));
    k_scan_blocksum<TI><<<(unsigned)nb, SB, 0, s>>>(in, n, bsum);
    MG_LAUNCH_CHECK();
    k_scan_bsums<<<1, SB, 0, s>>>(bsum, nb, out + n);
    MG_LAUNCH_CHECK();
    k_scan_final<TI><<<(unsigned)nb, SB, 0, s>>>(in, n, bsum, out);
    MG_LAUNCH_CHECK();
    MG_CK(cudaFreeAsync(bsum, s));
}
template void scan_exclusive<int32_t>(const int32_t*, int64_t*, int64_t, cudaStream_t);
template void scan_exclusive<int64_t>(const int64_t*, int64_t*, int64_t, cudaStream_t);
template void scan_exclusive<uint8_t>(const uint8_t*, int64_t*, int64_t, cudaStream_t);

namespace {
__global__ void k_finalize_sum(const double* parts, int np, double* out) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += 1024) v += parts[i];
    v = block_sum<1024>(v, sh);
    if (threadIdx.x == 0) *out = v;
}
__global__ void k_finalize_max(const double* parts, int np, double* out) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += 1024) v = fmax(v, parts[i]);
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = sh[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) *out = v;
    }
}
template <class A, class B>
__global__ void k_convert(const A* in, B* out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (B)in[i];
}
__global__ void k_fill_i32(int32_t* p, int32_t v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_iota_i32(int32_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = (int32_t)i;
}
__global__ void k_sort_segments(const int64_t* ptr, int32_t* keys, int64_t nseg) {
    int64_t sgi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sgi >= nseg) return;
    int64_t b = ptr[sgi], e = ptr[sgi + 1];
    for (int64_t i = b + 1; i < e; ++i) {
        int32_t k = keys[i];
        int64_t j = i - 1;
        while (j >= b && keys[j] > k) { keys[j + 1] = keys[j]; --j; }
        keys[j + 1] = k;
    }
}
__global__ void k_count_keys(const int32_t* key, int64_t n, int32_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[key[i]], 1);
}
__global__ void k_fill_keys(const int32_t* key, int64_t n, const int64_t* ptr, int32_t* cur, int32_t* list) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t k = key[i];
        int32_t pos = atomicAdd(&cur[k], 1);
        list[ptr[k] + pos] = (int32_t)i;
    }
}
inline int grid_for(int64_t n) { int64_t g = (n + 255) / 256; return (int)(g < 148 * 32 ? (g > 0 ? g : 1) : 148 * 32); }
}  // namespace

void finalize_sum(const double* parts, int np, double* out, cudaStream_t s) {
    k_finalize_sum<<<1, 1024, 0, s>>>(parts, np, out);
    MG_LAUNCH_CHECK();
}
void finalize_max(const double* parts, int np, double* out, cudaStream_t s) {
    k_finalize_max<<<1, 1024, 0, s>>>(parts, np, out);
    MG_LAUNCH_CHECK();
}
template <class A, class B>
void convert(const A* in, B* out, int64_t n, cudaStream_t s) {
    if (!n) return;
    k_convert<A, B><<<grid_for(n), 256, 0, s>>>(in, out, n);
    MG_LAUNCH_CHECK();
}
template void convert<double, float>(const double*, float*, int64_t, cudaStream_t);
template void convert<double, double>(const double*, double*, int64_t, cudaStream_t);
template void convert<float, double>(const float*, double*, int64_t, cudaStream_t);
template void convert<float, float>(const float*, float*, int64_t, cudaStream_t);

void fill_i32(int32_t* p, int32_t v, int64_t n, cudaStream_t s) {
    if (!n) return;
    k_fill_i32<<<grid_for(n), 256, 0, s>>>(p, v, n);
    MG_LAUNCH_CHECK();
}
void iota_i32(int32_t* p, int64_t n, cudaStream_t s) {
    if (!n) return;
    k_iota_i32<<<grid_for(n), 256, 0, s>>>(p, n);
    MG_LAUNCH_CHECK();
}
void sort_segments_i32(const int64_t* ptr, int32_t* keys, int64_t nseg, cudaStream_t s) {
    if (!nseg) return;
    k_sort_segments<<<ceil_div(nseg, 128), 128, 0, s>>>(ptr, keys, nseg);
    MG_LAUNCH_CHECK();
}
void group_by_key(const int32_t* key, int64_t n, int64_t nk, DBuf<int64_t>& ptr, DBuf<int32_t>& list,
                  DBuf<int32_t>& cnt, cudaStream_t s, bool sort) {
    ptr.resize(nk + 1);
    list.resize(n);
    cnt.resize(nk);
    MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (nk ? nk : 1), s));
    if (n) { k_count_keys<<<grid_for(n), 256, 0, s>>>(key, n, cnt.p); MG_LAUNCH_CHECK(); }
    scan_exclusive<int32_t>(cnt.p, ptr.p, nk, s);
    MG_CK(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (nk ? nk : 1), s));
    if (n) { k_fill_keys<<<grid_for(n), 256, 0, s>>>(key, n, ptr.p, cnt.p, list.p); MG_LAUNCH_CHECK(); }
    if (sort) sort_segments_i32(ptr.p, list.p, nk, s);
}

__global__ void k_stamp(unsigned long long* buf, int idx) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    buf[idx] = t;
}
void stamp(unsigned long long* buf, int idx, cudaStream_t s) {
    k_stamp<<<1, 1, 0, s>>>(buf, idx);
    MG_LAUNCH_CHECK();
}

// Raise (never lower) a kernel's dynamic shared-memory limit on the current device.  The cache is keyed
// by (device, kernel): the attribute is per device, and lowering it would break another live context
// that launches the same kernel with a larger plan.  Returns false (no throw) when `bytes` cannot be
// granted.
static bool raise_dyn_smem(const void* kernel, size_t bytes, bool throw_on_error) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;
    int dev = 0;
    MG_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[{dev, kernel}];
    if (bytes > cur && bytes > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) {
            if (throw_on_error) MG_CK(e);
            (void)cudaGetLastError();
            return false;
        }
        cur = bytes;
    }
    return true;
}
void ensure_dyn_smem(const void* kernel, size_t bytes) { raise_dyn_smem(kernel, bytes, true); }
bool try_raise_dyn_smem(const void* kernel, size_t bytes) { return raise_dyn_smem(kernel, bytes, false); }

}  // namespace mgpbd
