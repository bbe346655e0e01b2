// Deterministic scans / reductions / small vector kernels used by setup and solve.
#pragma once
#include "common.cuh"

namespace mgpbd {

// out[0..n] = exclusive prefix sum of in[0..n-1] (out[n] = total).  in may be int32 or int64.
template <class TI>
void scan_exclusive(const TI* in, int64_t* out, int64_t n, cudaStream_t s);

// out[slot] = sum of parts[0..np-1] in fixed order (single block).
void finalize_sum(const double* parts, int np, double* out, cudaStream_t s);
// out = max of parts (non-negative)
void finalize_max(const double* parts, int np, double* out, cudaStream_t s);

// Host-side convenience: read one device scalar (synchronises the stream).
template <class T>
T read_scalar(const T* d, cudaStream_t s) {
    T h;
    MG_CK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
    MG_CK(cudaStreamSynchronize(s));
    return h;
}

template <class A, class B>
void convert(const A* in, B* out, int64_t n, cudaStream_t s);

void fill_i32(int32_t* p, int32_t v, int64_t n, cudaStream_t s);
void iota_i32(int32_t* p, int64_t n, cudaStream_t s);

// segment-wise ascending sort of int32 keys (thread per segment, insertion sort; short segments)
void sort_segments_i32(const int64_t* ptr, int32_t* keys, int64_t nseg, cudaStream_t s);

// counting sort helper: given key[i] in [0,nk), build ptr (nk+1) and list (n) grouped by key with
// ascending i inside each group (deterministic).
void group_by_key(const int32_t* key, int64_t n, int64_t nk, DBuf<int64_t>& ptr, DBuf<int32_t>& list,
                  DBuf<int32_t>& tmp_cnt, cudaStream_t s, bool sort = true);

// Raise a kernel's dynamic shared-memory limit to at least `bytes` (thread-safe: contexts of virtual
// ranks launch from several host threads; the attribute is only ever raised).
void ensure_dyn_smem(const void* kernel, size_t bytes);      // raise-only, per (device, kernel); throws
bool try_raise_dyn_smem(const void* kernel, size_t bytes);   // same, returns false instead of throwing

// Diagnostics: buf[idx] = %globaltimer (one thread; graph-capturable; MGPBD_TRACE_STAGES).
void stamp(unsigned long long* buf, int idx, cudaStream_t s);

}  // namespace mgpbd
