// common.cuh — element types, 16-byte vector access and warp shuffles shared by
// the sm_100a stencil kernels.  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace stb200 {

constexpr unsigned FULL = 0xffffffffu;

// One lane owns one 16-byte vector of a warp row tile: V elements of T
// (float4 / int4 for 32-bit types, double2 for fp64).  A warp therefore owns
// 512 contiguous bytes of a row: 128 fp32/int32 points or 64 fp64 points.
template <typename T> struct VecOf;
template <> struct VecOf<float>   { using type = float4;  static constexpr int V = 4; };
template <> struct VecOf<int>     { using type = int4;    static constexpr int V = 4; };
template <> struct VecOf<double>  { using type = double2; static constexpr int V = 2; };

template <typename T> constexpr int vlen() { return VecOf<T>::V; }

// 16-byte read-only load (LDG.E.128.CONSTANT) into v[0..V).
template <typename T>
__device__ __forceinline__ void ldg_vec(T* v, const T* p) {
    using VT = typename VecOf<T>::type;
    const VT t = __ldg(reinterpret_cast<const VT*>(p));
    if constexpr (VecOf<T>::V == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
    else { v[0] = t.x; v[1] = t.y; }
}

// 16-byte store (STG.E.128).
template <typename T>
__device__ __forceinline__ void stg_vec(T* p, const T* v) {
    using VT = typename VecOf<T>::type;
    VT t;
    if constexpr (VecOf<T>::V == 4) { t.x = v[0]; t.y = v[1]; t.z = v[2]; t.w = v[3]; }
    else { t.x = v[0]; t.y = v[1]; }
    *reinterpret_cast<VT*>(p) = t;
}

// 16-byte shared-memory store (STS.128).
template <typename T>
__device__ __forceinline__ void st_vec_s(T* p, const T* v) { stg_vec(p, v); }

// 16-byte streaming store (st.global.cs: evict-first in L1/L2).
template <typename T>
__device__ __forceinline__ void stcs_vec(T* p, const T* v) {
    using VT = typename VecOf<T>::type;
    VT t;
    if constexpr (VecOf<T>::V == 4) { t.x = v[0]; t.y = v[1]; t.z = v[2]; t.w = v[3]; }
    else { t.x = v[0]; t.y = v[1]; }
    __stcs(reinterpret_cast<VT*>(p), t);
}

// Load R consecutive elements starting at p; p is aligned to R*sizeof(T)
// whenever R*sizeof(T) is 8 or 16 (see the alignment argument in k2d.cuh).
template <typename T, int R>
__device__ __forceinline__ void ldg_run(T* v, const T* p) {
    if constexpr (R == 2 && std::is_same<T, float>::value) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p)); v[0] = t.x; v[1] = t.y;
    } else if constexpr (R == 2 && std::is_same<T, int>::value) {
        const int2 t = __ldg(reinterpret_cast<const int2*>(p)); v[0] = t.x; v[1] = t.y;
    } else if constexpr (R == 2 && sizeof(T) == 8) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p)); v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = __ldg(p + k);
    }
}

// Predicated shared-memory load of R consecutive elements into dst (dst is
// left unchanged where the predicate is false): the corner-lane fallback
// without a select.  The address is R*sizeof(T)-aligned at every call site.
template <typename T, int R>
__device__ __forceinline__ void lds_pred(bool p, const T* src, T* dst) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(src));
    const int pi = p ? 1 : 0;
    if constexpr (std::is_same<T, float>::value && R == 2) {
        asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.f32 {%0, %1}, [%3];}"
                     : "+f"(dst[0]), "+f"(dst[1]) : "r"(pi), "r"(a));
    } else if constexpr (std::is_same<T, float>::value && R == 1) {
        asm volatile("{.reg .pred q; setp.ne.b32 q, %1, 0; @q ld.shared.f32 %0, [%2];}"
                     : "+f"(dst[0]) : "r"(pi), "r"(a));
    } else if constexpr (std::is_same<T, int>::value && R == 2) {
        asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.b32 {%0, %1}, [%3];}"
                     : "+r"(dst[0]), "+r"(dst[1]) : "r"(pi), "r"(a));
    } else if constexpr (std::is_same<T, int>::value && R == 1) {
        asm volatile("{.reg .pred q; setp.ne.b32 q, %1, 0; @q ld.shared.b32 %0, [%2];}"
                     : "+r"(dst[0]) : "r"(pi), "r"(a));
    } else if constexpr (std::is_same<T, double>::value && R == 2) {
        asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.f64 {%0, %1}, [%3];}"
                     : "+d"(dst[0]), "+d"(dst[1]) : "r"(pi), "r"(a));
    } else {
        asm volatile("{.reg .pred q; setp.ne.b32 q, %1, 0; @q ld.shared.f64 %0, [%2];}"
                     : "+d"(dst[0]) : "r"(pi), "r"(a));
    }
}

// Shuffles move 32-bit patterns unchanged (PAPER.md:272-274 restricts the
// paper to 32-bit data); a 64-bit element is two SHFL.
__device__ __forceinline__ float  shfl_up(float v, int d)   { return __shfl_up_sync(FULL, v, d); }
__device__ __forceinline__ int    shfl_up(int v, int d)     { return __shfl_up_sync(FULL, v, d); }
__device__ __forceinline__ double shfl_up(double v, int d)  { return __shfl_up_sync(FULL, v, d); }
__device__ __forceinline__ float  shfl_down(float v, int d) { return __shfl_down_sync(FULL, v, d); }
__device__ __forceinline__ int    shfl_down(int v, int d)   { return __shfl_down_sync(FULL, v, d); }
__device__ __forceinline__ double shfl_down(double v, int d){ return __shfl_down_sync(FULL, v, d); }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Fused halo exchange (dist.cu P2P transport): the output planes/rows a
// neighbour rank needs as halo are also stored straight into its buffer
// through a peer pointer.  Slow-axis index q < lo_end goes to `lo` at element
// offset + d_lo; q >= hi_begin goes to `hi` at offset + d_hi.  Null = off.
template <typename T> struct PeerOut {
    T* lo = nullptr;
    T* hi = nullptr;
    int64_t lo_end = 0, hi_begin = 0, d_lo = 0, d_hi = 0;
};

// Coefficients passed by value as a kernel parameter (constant bank): FFMA
// reads them as c[bank][offset] operands, no registers spent.
template <typename T, int N> struct Coeffs { T c[N > 0 ? N : 1]; };

}  // namespace stb200
