// Vector loads of one constraint's vertex ids and scaled-gradient record h (KC slots x 3 values,
// storage precision T): shared by the assembly and the matrix-free level-0 operator.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace mgpbd {

__device__ __forceinline__ void load_iv(const int4& v, int (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
__device__ __forceinline__ void load_iv(const int2& v, int (&o)[2]) { o[0] = v.x; o[1] = v.y; }

// one constraint's scaled-gradient record (KC slots x 3) with 16-/8-byte vector loads
template <class T, int KC>
__device__ __forceinline__ void load_record(const T* __restrict__ p, T (&o)[KC][3]) {
    constexpr int N = KC * 3;
    T tmp[N];
    if constexpr (sizeof(T) == 4 && KC == 4) {
        const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float4 v = q[k];
            tmp[4 * k] = v.x; tmp[4 * k + 1] = v.y; tmp[4 * k + 2] = v.z; tmp[4 * k + 3] = v.w;
        }
    } else {
        using V2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
        const V2* q = reinterpret_cast<const V2*>(p);
#pragma unroll
        for (int k = 0; k < N / 2; ++k) {
            const V2 v = q[k];
            tmp[2 * k] = v.x; tmp[2 * k + 1] = v.y;
        }
    }
#pragma unroll
    for (int k = 0; k < KC; ++k)
#pragma unroll
        for (int r = 0; r < 3; ++r) o[k][r] = tmp[3 * k + r];
}

}  // namespace mgpbd
