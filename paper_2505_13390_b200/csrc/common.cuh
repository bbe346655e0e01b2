// Shared device/host utilities of libmgpbd (CUDA path only; nothing here is used by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <utility>
#include <string>
#include <vector>

namespace mgpbd {

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define MG_CK(call)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            throw ::mgpbd::Error(e_ == cudaErrorMemoryAllocation ? -4 : -2,                      \
                                 std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +     \
                                     __FILE__ + ":" + std::to_string(__LINE__));                 \
    } while (0)

// Every kernel launch site is followed by exactly one MG_LAUNCH_CHECK(): it counts the launch
// (reported as mgpbd_stats.kernel_launches) and surfaces launch errors.
extern thread_local int64_t g_kernel_launches;
#define MG_LAUNCH_CHECK()                 \
    do {                                  \
        ++::mgpbd::g_kernel_launches;     \
        MG_CK(cudaGetLastError());        \
    } while (0)

constexpr int kWarp = 32;

// Stream on which the current thread's context allocates (stream-ordered allocation from the
// device's default memory pool, whose release threshold the context raises so that setup-time
// temporaries are recycled instead of being mapped/unmapped every setup).  nullptr = cudaMalloc.
extern thread_local cudaStream_t g_alloc_stream;

inline void dev_free(void* p) {
    if (!p) return;
    if (g_alloc_stream) cudaFreeAsync(p, g_alloc_stream);
    else cudaFree(p);
}

// Growable device buffer (owns memory; never shrinks).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { dev_free(p); }
    void resize(size_t m) {
        if (m > cap) {
            dev_free(p);
            p = nullptr;
            // +16 elements: vectorised streams may read up to one 32-byte vector past the end
            if (g_alloc_stream) MG_CK(cudaMallocAsync(&p, (m + 16) * sizeof(T), g_alloc_stream));
            else MG_CK(cudaMalloc(&p, (m + 16) * sizeof(T)));
            cap = m;
        }
        n = m;
    }
    void swap(DBuf& o) { std::swap(p, o.p); std::swap(n, o.n); std::swap(cap, o.cap); }
    void free_all() { dev_free(p); p = nullptr; n = cap = 0; }
    T* get() const { return p; }
    size_t bytes() const { return n * sizeof(T); }
};

template <class T>
inline void h2d(T* d, const T* h, size_t n, cudaStream_t s) {
    if (n) MG_CK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
inline void d2h(T* h, const T* d, size_t n, cudaStream_t s) {
    if (n) MG_CK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}
template <class T>
inline void d2d(T* d, const T* s_, size_t n, cudaStream_t s) {
    if (n) MG_CK(cudaMemcpyAsync(d, s_, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------- device helpers
// splitmix64 finaliser and the keyed hash of reading c0: key(stream,l,i) =
// mix64(mix64(seed ^ stream<<56 ^ l<<48) ^ i); U = ((key>>11)+0.5) 2^-53.
__host__ __device__ __forceinline__ uint64_t hmix(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}
__host__ __device__ __forceinline__ uint64_t hkey_base(uint64_t seed, int stream, int level) {
    return hmix(seed ^ ((uint64_t)stream << 56) ^ ((uint64_t)level << 48));
}
__host__ __device__ __forceinline__ uint64_t hkey(uint64_t base, uint64_t i) { return hmix(base ^ i); }
__host__ __device__ __forceinline__ double hunit(uint64_t key) {
    return ((double)(key >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

// Fixed-order sub-warp sum (butterfly within groups of VL lanes): identical result in every lane.
template <int VL>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = VL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, VL);
    return v;
}

template <int VL, class U>
__device__ __forceinline__ U group_sum_t(U v) {
#pragma unroll
    for (int o = VL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, VL);
    return v;
}

// Deterministic block sum of per-thread values (fixed tree); result valid in thread 0.
template <int BS>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = group_sum<32>(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < BS / 32) ? sh[l] : 0.0;
        r = group_sum<32>(r);
    }
    __syncthreads();
    return r;
}

}  // namespace mgpbd
