// kpaper3d.cuh — the paper-literal variant family (kpaper.cuh, SURVEY §8(f)
// row f1) for the 3-D suite members: laplacian, wave13pt, divergence,
// gradient, tricubic (fp32: the paper shuffles 32-bit data).
//
// One output point per thread; threads along x (the leading dimension,
// `vector(512)` of Listing 5), blocks over (x blocks, rows y, planes z).
// Every x-row of taps (fixed array, dz, dy) with more than one x tap is
// shuffle-synthesised the way PTXASW does it: the leftmost tap is the
// source load, every other tap of the row is a destination at delta
// N = dx - dx_min (shfl.sync.down) with the Listing 6 corner fallback; taps
// alone in their row stay loads.  This reproduces Table 1:
//   laplacian  x-row {-1,0,1}            2 shuffles / 7 loads,  delta 1.5
//   wave13pt   x-row {-2..2} of cur      4 / 14 (13 + prev),    delta 2.5
//   divergence x-row {-1,+1} of u        1 / 6,                 delta 2.0
//   gradient   x-row {-1,+1}             1 / 6,                 delta 2.0
//   tricubic   16 x-rows {-1..2} of f    48 / 67 (64 + X,Y,Z),  delta 2.0
// The point formulas use the register-cache kernels' term order (k3d.cuh
// Op::point) so ORIGINAL / PTXASW / UNIFORM are bit-identical to SHUFFLE for
// the k3d kinds; tricubic follows the oracle's Lagrange form and order.
#pragma once
#include "kpaper.cuh"

namespace stb200 {

// Taps of one x-row: t[q] = row[(Lo + q*STEP)] for q = 0..NT-1; tap 0 is the
// source load, tap q a destination at shuffle delta q*STEP.
template <int Lo, int NT, int STEP, int PV, bool COMPLETE>
__device__ __forceinline__ void xrow(const uint32_t* p, uint32_t* t) {
    const uint32_t src = ldg_nc_b32(p + Lo);
    t[0] = src;
    if constexpr (NT > 1) t[1] = dest_n<1 * STEP, PV, COMPLETE>(src, p + Lo + 1 * STEP);
    if constexpr (NT > 2) t[2] = dest_n<2 * STEP, PV, COMPLETE>(src, p + Lo + 2 * STEP);
    if constexpr (NT > 3) t[3] = dest_n<3 * STEP, PV, COMPLETE>(src, p + Lo + 3 * STEP);
    if constexpr (NT > 4) t[4] = dest_n<4 * STEP, PV, COMPLETE>(src, p + Lo + 4 * STEP);
}

__device__ __forceinline__ float ldf(const uint32_t* p) { return __uint_as_float(ldg_nc_b32(p)); }
__device__ __forceinline__ float bf(uint32_t b) { return __uint_as_float(b); }

// KIND: 1 laplacian3d7 / jacobi3d7, 2 wave13pt, 3 divergence, 4 gradient, 5 tricubic
struct P3Args {
    const uint32_t* in[4];
    float* out[3];
    int64_t nx, ny;
    int z_lo, lo, hi;
    float c[3];
};

template <int KIND, int PV, bool COMPLETE>
__device__ __forceinline__ void p3_point(const P3Args& a, int64_t o, int64_t sy, int64_t sz) {
    if constexpr (KIND == 1) {                             // a*C + b*(x+1 + x-1 + y+1 + y-1 + z+1 + z-1)
        const uint32_t* u = a.in[0] + o;
        uint32_t x[3];
        xrow<-1, 3, 1, PV, COMPLETE>(u, x);
        float s = bf(x[2]) + bf(x[0]);
        s = s + ldf(u + sy);
        s = s + ldf(u - sy);
        s = s + ldf(u + sz);
        s = s + ldf(u - sz);
        a.out[0][o] = fmaf(a.c[1], s, a.c[0] * bf(x[1]));
    } else if constexpr (KIND == 2) {                      // leapfrog 13-point (prev, cur) -> next
        const uint32_t* u = a.in[1] + o;
        uint32_t x[5];
        xrow<-2, 5, 1, PV, COMPLETE>(u, x);
        float s1 = bf(x[3]) + bf(x[1]);
        s1 = s1 + ldf(u + sy);
        s1 = s1 + ldf(u - sy);
        s1 = s1 + ldf(u + sz);
        s1 = s1 + ldf(u - sz);
        float s2 = bf(x[4]) + bf(x[0]);
        s2 = s2 + ldf(u + 2 * sy);
        s2 = s2 + ldf(u - 2 * sy);
        s2 = s2 + ldf(u + 2 * sz);
        s2 = s2 + ldf(u - 2 * sz);
        float r = fmaf(a.c[1], s1, a.c[0] * bf(x[2]));
        r = fmaf(a.c[2], s2, r);
        a.out[0][o] = r - ldf(a.in[0] + o);
    } else if constexpr (KIND == 3) {                      // ax(u x+1 - x-1) + ay(v ..) + az(w ..)
        uint32_t x[2];
        xrow<-1, 2, 2, PV, COMPLETE>(a.in[0] + o, x);
        float r = a.c[0] * (bf(x[1]) - bf(x[0]));
        r = fmaf(a.c[1], ldf(a.in[1] + o + sy) - ldf(a.in[1] + o - sy), r);
        a.out[0][o] = fmaf(a.c[2], ldf(a.in[2] + o + sz) - ldf(a.in[2] + o - sz), r);
    } else if constexpr (KIND == 4) {                      // (ax(x+1 - x-1), ay(..), az(..))
        const uint32_t* u = a.in[0] + o;
        uint32_t x[2];
        xrow<-1, 2, 2, PV, COMPLETE>(u, x);
        a.out[0][o] = a.c[0] * (bf(x[1]) - bf(x[0]));
        a.out[1][o] = a.c[1] * (ldf(u + sy) - ldf(u - sy));
        a.out[2][o] = a.c[2] * (ldf(u + sz) - ldf(u - sz));
    } else {                                               // tricubic (oracle form and order)
        float w[3][4];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const float t = ldf(a.in[1 + d] + o);
            w[d][0] = -t * (t - 1.f) * (t - 2.f) / 6.f;
            w[d][1] = (t + 1.f) * (t - 1.f) * (t - 2.f) / 2.f;
            w[d][2] = -(t + 1.f) * t * (t - 2.f) / 2.f;
            w[d][3] = (t + 1.f) * t * (t - 1.f) / 6.f;
        }
        float g = 0.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            float sb = 0.f;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                uint32_t x[4];
                xrow<-1, 4, 1, PV, COMPLETE>(a.in[0] + o + (cc - 1) * sz + (b - 1) * sy, x);
                float sa = w[0][0] * bf(x[0]);
#pragma unroll
                for (int q = 1; q < 4; ++q) sa = sa + w[0][q] * bf(x[q]);
                sb = b == 0 ? w[1][0] * sa : sb + w[1][b] * sa;
            }
            g = cc == 0 ? w[2][0] * sb : g + w[2][cc] * sb;
        }
        a.out[0][o] = g;
    }
}

// Grid: x = ceil((nx - lo - hi) / 512), y = interior rows, z = output planes.
template <int KIND, int PV>
__global__ void __launch_bounds__(kPaperThreads) kpaper3d(const __grid_constant__ P3Args a) {
    const int64_t i = a.lo + (int64_t)blockIdx.x * kPaperThreads + threadIdx.x;
    if (i >= a.nx - a.hi) return;                          // the last warp of a row is incomplete
    const int64_t j = a.lo + blockIdx.y;
    const int64_t k = a.z_lo + blockIdx.z;
    const int64_t sy = a.nx, sz = a.nx * a.ny;
    const int64_t o = k * sz + j * sy + i;
    if constexpr (PV == PV_UNIFORM) {
        if (__activemask() == FULL) p3_point<KIND, PV, true>(a, o, sy, sz);
        else p3_point<KIND, PV, false>(a, o, sy, sz);
    } else {
        p3_point<KIND, PV, true>(a, o, sy, sz);
    }
}

}  // namespace stb200
