// kpaper.cuh — the paper's own code shape on B200:
// one output point per thread, threads along the leading dimension, and the
// PTXASW transformation of Listing 6 written out in
// inline PTX, plus the paper's ablations and the
// uniform-branch variant of its Pascal analysis.
//
// Launch shape follows Listing 5: `gang` over rows j (grid
// y), `vector(512)` over columns i (512 threads per block along x).  Threads
// past the row end exit, so the last warp of a row is incomplete — the
// paper's %incomplete corner case.
//
// Per x-row of taps (row offset dj) the leftmost tap is the source load
// (ld.global.nc); every other tap di > -R of that row is a destination at
// shuffle delta N = di + R > 0 (shfl.sync.down: lane l receives lane l+N;
// PAPER.md:509, 565).  Table 1's counts follow (jacobi 6/9, delta 1.5;
// gaussblur 20/25, delta 2.5; gameoflife 6/9, delta 1.5).
//
// Variants (ST_PAPER_*):
//   ORIGINAL   every tap is its own ld.global.nc (the compiler's code)
//   PTXASW     Listing 6: source mov; activemask; %incomplete = mask != ~0;
//              %out_of_range = laneid > 31-N; or.pred; shfl.sync.down at the
//              load site; @%pred the original load (no new branch, no select)
//   NOLOAD     covered loads removed (destinations reuse the source value):
//              invalid results, the memory-instruction upper bound
//   NOCORNER   shuffles without the corner fallback: invalid at warp edges
//   UNIFORM    warp-uniform branch: complete warps take shuffles with the
//              out-of-range fallback, incomplete warps take ORIGINAL loads
#pragma once
#include "common.cuh"

namespace stb200 {

enum { PV_ORIGINAL = 0, PV_PTXASW = 1, PV_NOLOAD = 2, PV_NOCORNER = 3, PV_UNIFORM = 4 };

__device__ __forceinline__ uint32_t ldg_nc_b32(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// One destination tap of Listing 6: shuffle `src` down by N with the
// predicated original load as the corner fallback.
template <int N>
__device__ __forceinline__ uint32_t ptxasw_dest(uint32_t src, const void* addr) {
    uint32_t d;
    asm volatile(
        "{\n\t"
        ".reg .b32 mask, lane, srcc;\n\t"
        ".reg .pred incomplete, out_of_range, pred;\n\t"
        "mov.b32 srcc, %1;\n\t"                                   // source register
        "activemask.b32 mask;\n\t"
        "setp.ne.u32 incomplete, mask, 0xffffffff;\n\t"
        "mov.u32 lane, %%laneid;\n\t"
        "setp.gt.u32 out_of_range, lane, %3;\n\t"
        "or.pred pred, incomplete, out_of_range;\n\t"
        "shfl.sync.down.b32 %0, srcc, %4, 31, mask;\n\t"
        "@pred ld.global.nc.b32 %0, [%2];\n\t"
        "}"
        : "=r"(d)
        : "r"(src), "l"(addr), "n"(31 - N), "n"(N));
    return d;
}

template <int N>
__device__ __forceinline__ uint32_t nocorner_dest(uint32_t src) {
    uint32_t d;
    asm volatile(
        "{\n\t.reg .b32 mask;\n\t"
        "activemask.b32 mask;\n\t"
        "shfl.sync.down.b32 %0, %1, %2, 31, mask;\n\t}"
        : "=r"(d)
        : "r"(src), "n"(N));
    return d;
}

// Out-of-range-only form used by the UNIFORM variant inside a complete warp.
template <int N>
__device__ __forceinline__ uint32_t uniform_dest(uint32_t src, const void* addr) {
    uint32_t d;
    asm volatile(
        "{\n\t.reg .b32 lane;\n\t.reg .pred out_of_range;\n\t"
        "mov.u32 lane, %%laneid;\n\t"
        "setp.gt.u32 out_of_range, lane, %3;\n\t"
        "shfl.sync.down.b32 %0, %1, %4, 31, 0xffffffff;\n\t"
        "@out_of_range ld.global.nc.b32 %0, [%2];\n\t}"
        : "=r"(d)
        : "r"(src), "l"(addr), "n"(31 - N), "n"(N));
    return d;
}

template <typename T> __device__ __forceinline__ T from_bits(uint32_t b);
template <> __device__ __forceinline__ float from_bits<float>(uint32_t b) { return __uint_as_float(b); }
template <> __device__ __forceinline__ int from_bits<int>(uint32_t b) { return (int)b; }

template <int N, int PV, bool COMPLETE>
__device__ __forceinline__ uint32_t dest_n(uint32_t src, const void* a) {
    if constexpr (PV == PV_ORIGINAL) return ldg_nc_b32(a);
    else if constexpr (PV == PV_NOLOAD) return src;
    else if constexpr (PV == PV_NOCORNER) return nocorner_dest<N>(src);
    else if constexpr (PV == PV_UNIFORM) return COMPLETE ? uniform_dest<N>(src, a) : ldg_nc_b32(a);
    else return ptxasw_dest<N>(src, a);
}

// Taps of one row (dj) for the thread's point i: t[di + R] = in[j+dj][i+di].
template <int R, int PV, bool COMPLETE>
__device__ __forceinline__ void row_taps(const uint32_t* rowp, uint32_t* t) {
    const uint32_t src = ldg_nc_b32(rowp - R);                   // source: leftmost tap
    t[0] = src;
    t[1] = dest_n<1, PV, COMPLETE>(src, rowp - R + 1);            // N = di + R
    t[2] = dest_n<2, PV, COMPLETE>(src, rowp - R + 2);
    if constexpr (R >= 2) {
        t[3] = dest_n<3, PV, COMPLETE>(src, rowp - R + 3);
        t[4] = dest_n<4, PV, COMPLETE>(src, rowp - R + 4);
    }
}

// Point formulas (same term order as k2d.cuh / the oracle).
template <typename T, int KIND> struct PaperOp;
template <typename T> struct PaperOp<T, 1> {            // jacobi2d5
    static constexpr int R = 1, NC = 2;
    __device__ static T f(const T (*w)[3], const Coeffs<T, NC>& c) {
        T s = w[1][0] + w[0][1];
        s = s + w[1][2];
        s = s + w[2][1];
        return fma(c.c[1], s, c.c[0] * w[1][1]);
    }
};
template <typename T> struct PaperOp<T, 2> {            // jacobi2d9
    static constexpr int R = 1, NC = 3;
    __device__ static T f(const T (*w)[3], const Coeffs<T, NC>& c) {
        T s1 = w[1][0] + w[0][1];
        s1 = s1 + w[1][2];
        s1 = s1 + w[2][1];
        T s2 = w[0][0] + w[2][0];
        s2 = s2 + w[0][2];
        s2 = s2 + w[2][2];
        T r = fma(c.c[1], s1, c.c[0] * w[1][1]);
        return fma(c.c[2], s2, r);
    }
};
template <typename T> struct PaperOp<T, 3> {            // gaussblur5x5
    static constexpr int R = 2, NC = 25;
    __device__ static T f(const T (*w)[5], const Coeffs<T, NC>& c) {
        T acc = c.c[0] * w[0][0];
#pragma unroll
        for (int t = 1; t < 25; ++t) acc = fma(c.c[t], w[t / 5][t % 5], acc);
        return acc;
    }
};
template <typename T> struct PaperOp<T, 4> {            // gameoflife
    static constexpr int R = 1, NC = 0;
    __device__ static int f(const int (*w)[3], const Coeffs<T, NC>&) {
        const int n = w[0][0] + w[0][1] + w[0][2] + w[1][0] + w[1][2] + w[2][0] + w[2][1] + w[2][2];
        return (n == 3 || (n == 2 && w[1][1] == 1)) ? 1 : 0;
    }
};

constexpr int kPaperThreads = 512;                       // Listing 5: vector(512)

// Grid: x = ceil((nx - 2R) / 512) column blocks, y = output rows [y_lo, y_hi).
template <typename T, int KIND, int PV>
__global__ void __launch_bounds__(kPaperThreads)
kpaper(const T* __restrict__ in, T* __restrict__ out, int64_t nx, int y_lo,
       Coeffs<T, PaperOp<T, KIND>::NC> c) {
    using Op = PaperOp<T, KIND>;
    constexpr int R = Op::R, D = 2 * R + 1;
    const int64_t j = y_lo + blockIdx.y;
    const int64_t i = R + (int64_t)blockIdx.x * kPaperThreads + threadIdx.x;
    if (i >= nx - R) return;                               // the last warp becomes incomplete
    const uint32_t* base = reinterpret_cast<const uint32_t*>(in) + j * nx + i;
    uint32_t t[D][D];
    if constexpr (PV == PV_UNIFORM) {
        if (__activemask() == FULL) {                      // warp-uniform branch (!%incomplete)
#pragma unroll
            for (int dj = -R; dj <= R; ++dj) row_taps<R, PV, true>(base + dj * nx, t[dj + R]);
        } else {
#pragma unroll
            for (int dj = -R; dj <= R; ++dj) row_taps<R, PV, false>(base + dj * nx, t[dj + R]);
        }
    } else {
#pragma unroll
        for (int dj = -R; dj <= R; ++dj) row_taps<R, PV, true>(base + dj * nx, t[dj + R]);
    }
    T w[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) w[a][b] = from_bits<T>(t[a][b]);
    out[j * nx + i] = Op::f(w, c);
}

}  // namespace stb200
