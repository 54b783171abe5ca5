// k2d.cuh — 2-D register-cache stencil kernels for sm_100a.
//
// The paper's transformation (§5, 503-576) turns a load of a
// neighbour element that an adjacent thread already loaded into a warp
// shuffle, A(tid+N) = B(tid) with -31 <= N <= 31, with a
// predicated original load as the corner-case fallback.
// On B200 the 1-output-per-thread form of that idea cannot reach the HBM
// roofline (20 SHFL or 25 loads per point for gaussblur), so
// the kernels here are register-blocked first and shuffle second:
//
//  * S1 map: a warp owns one x-tile of 32 lanes x V elements (one 16-byte
//    vector per lane: 128 fp32/int32 or 64 fp64 points) and marches down a
//    strip of H rows (the slow axis y).  A CTA holds kWarps2D adjacent
//    x-tiles of the same strip, so warp-edge fallback loads hit L1.
//  * S2 row-tile load: one coalesced LDG.128 per lane per row, issued D rows
//    ahead into a register ring of NS = 2R+1+D rows (software pipeline).
//  * S3 x-neighbour taps: the R elements left / right of a lane's vector.
//      SHUFFLE: shfl.sync.up/down by one lane (N = -1 / +1 in lane units).
//      PLAIN:   loads of the same elements (L1-resident: the neighbour lane
//               loaded that line in the same instruction).
//  * S4 corner cases: lane 0 / lane 31 take their outer halo from a
//    predicated load (the %out_of_range fallback); lanes past the row end
//    clamp their address (the warp stays full, no %incomplete case) and
//    their stores are masked.  No branch is divergent except the store mask
//    in the two edge tiles of a row.
//  * S5 slow-axis taps: the ring keeps the 2R+1 rows of the y-window in
//    registers; a row is loaded from HBM exactly once per strip.
//  * S6 arithmetic: Op::point on the register window, identical code for
//    both variants (so SHUFFLE == PLAIN bit for bit).
//  * S7 store: STG.128 of interior points; the boundary ring is never
//    written.
#pragma once
#include "common.cuh"

namespace stb200 {

constexpr int kWarps2D = 4;       // x-tiles per CTA (128 threads)
constexpr int kDepth2D = 3;       // rows in flight per warp (prefetch distance)

enum { VAR_SHUFFLE = 0, VAR_PLAIN = 1 };

// Read-only view of the register window for output row y at unroll phase u:
// w(dj, e) = element e (0 .. V+2R-1, centre of output p at e = p+R) of input
// row y+dj.  All indices fold to constants after unrolling.
template <typename T, int NS, int W, int R>
struct Win {
    const T (&a)[NS][W];
    int u;
    __device__ __forceinline__ T operator()(int dj, int e) const { return a[(u + R + dj) % NS][e]; }
};

// ---------------------------------------------------------------- stencils
// Each Op gives the radius R, coefficient count NC and the point formula in
// the oracle's term order (oracle/oracle.c), evaluated in T with FMA.

// jacobi2d5: c0*C + c1*(W + N + E + S)  (Listing 5 without the c2 term)
template <typename T> struct OpJacobi2D5 {
    static constexpr int R = 1, NC = 2;
    template <class Wn>
    __device__ __forceinline__ static T point(const Wn& w, int p, const Coeffs<T, NC>& c) {
        const int e = p + R;
        T s = w(0, e - 1) + w(-1, e);
        s = s + w(0, e + 1);
        s = s + w(1, e);
        return fma(c.c[1], s, c.c[0] * w(0, e));
    }
};

// jacobi2d9: Listing 5
template <typename T> struct OpJacobi2D9 {
    static constexpr int R = 1, NC = 3;
    template <class Wn>
    __device__ __forceinline__ static T point(const Wn& w, int p, const Coeffs<T, NC>& c) {
        const int e = p + R;
        T s1 = w(0, e - 1) + w(-1, e);
        s1 = s1 + w(0, e + 1);
        s1 = s1 + w(1, e);
        T s2 = w(-1, e - 1) + w(1, e - 1);
        s2 = s2 + w(-1, e + 1);
        s2 = s2 + w(1, e + 1);
        T r = fma(c.c[1], s1, c.c[0] * w(0, e));
        return fma(c.c[2], s2, r);
    }
};

// gaussblur5x5: correlation, acc over dj then di (Table 1, 25 loads)
template <typename T> struct OpGauss5 {
    static constexpr int R = 2, NC = 25;
    template <class Wn>
    __device__ __forceinline__ static T point(const Wn& w, int p, const Coeffs<T, NC>& c) {
        T acc = c.c[0] * w(-2, p);
#pragma unroll
        for (int t = 1; t < 25; ++t) acc = fma(c.c[t], w(t / 5 - 2, p + t % 5), acc);
        return acc;
    }
};

// gameoflife: Conway B3/S23 on int cells (Table 1, 9 loads)
struct OpLife {
    static constexpr int R = 1, NC = 0;
    template <class Wn>
    __device__ __forceinline__ static int point(const Wn& w, int p, const Coeffs<int, NC>&) {
        const int e = p + R;
        const int n = w(-1, e - 1) + w(-1, e) + w(-1, e + 1) + w(0, e - 1) + w(0, e + 1)
                    + w(1, e - 1) + w(1, e) + w(1, e + 1);
        return (n == 3 || (n == 2 && w(0, e) == 1)) ? 1 : 0;
    }
};

// ------------------------------------------------------------------ kernel
// Grid: x = ceil(ntiles / kWarps2D), y = strips of H output rows covering
// output rows [y_lo, y_hi) (R <= y_lo, y_hi <= ny - R).
template <class Op, typename T, int VARIANT, int D = kDepth2D>
__global__ void __launch_bounds__(kWarps2D * 32)
k2d(const T* __restrict__ in, T* __restrict__ out, int64_t nx, int y_lo, int y_hi, int H,
    Coeffs<T, Op::NC> c) {
    constexpr int R = Op::R;
    constexpr int V = vlen<T>();
    constexpr int W = V + 2 * R;          // lane window width: halo | vector | halo
    constexpr int NS = 2 * R + 1 + D;     // register ring: y-window + rows in flight
    static_assert(R <= V, "halo wider than one lane vector");

    const int lane = lane_id();
    const int64_t x0 = ((int64_t)blockIdx.x * kWarps2D + (threadIdx.x >> 5)) * (32 * V);
    if (x0 >= nx) return;                                   // warp-uniform
    const int ys = y_lo + (int)blockIdx.y * H;
    const int ye = min(ys + H, y_hi);
    if (ys >= ye) return;
    const int row_end = ye + R;                            // rows [ys-R, ye+R) are read

    const int64_t xl = x0 + lane * V;                      // first column of this lane
    const bool own = xl < nx;
    const int64_t xr = own ? xl : nx - V;                  // clamped: the warp stays full
    const bool left_edge = lane == 0 && x0 - R >= 0;       // %out_of_range, N = -1
    const bool right_edge = lane == 31 && x0 + 32 * V < nx; // %out_of_range, N = +1

    T win[NS][W];

    auto load = [&](int s, int row) {                       // S2
        if (row < row_end) ldg_vec(&win[s][R], in + (int64_t)row * nx + xr);
    };
    auto finalize = [&](int s, int row) {                   // S3 + S4
        const T* rp = in + (int64_t)row * nx;
        if constexpr (VARIANT == VAR_SHUFFLE) {
#pragma unroll
            for (int k = 0; k < R; ++k) win[s][k] = shfl_up(win[s][V + k], 1);
#pragma unroll
            for (int k = 0; k < R; ++k) win[s][R + V + k] = shfl_down(win[s][R + k], 1);
            if (left_edge) ldg_run<T, R>(&win[s][0], rp + x0 - R);
            if (right_edge) ldg_run<T, R>(&win[s][R + V], rp + x0 + 32 * V);
        } else {
            if (xr - R >= 0) ldg_run<T, R>(&win[s][0], rp + xr - R);
            if (xr + V + R <= nx) ldg_run<T, R>(&win[s][R + V], rp + xr + V);
        }
    };

#pragma unroll
    for (int s = 0; s < NS; ++s) load(s, ys - R + s);
#pragma unroll
    for (int s = 0; s < 2 * R; ++s) finalize(s, ys - R + s);

    const bool vec_store = own && xl >= R && xl + V <= nx - R;
    for (int y0 = ys; y0 < ye; y0 += NS) {
#pragma unroll
        for (int u = 0; u < NS; ++u) {
            const int y = y0 + u;
            if (y < ye) {                                   // warp-uniform
                finalize((u + 2 * R) % NS, y + R);
                T o[V];
                const Win<T, NS, W, R> w{win, u};
#pragma unroll
                for (int p = 0; p < V; ++p) o[p] = Op::point(w, p, c);   // S6
                T* orow = out + (int64_t)y * nx;
                if (vec_store) {
                    stg_vec(orow + xl, o);                              // S7
                } else if (own) {
#pragma unroll
                    for (int p = 0; p < V; ++p)
                        if (xl + p >= R && xl + p < nx - R) orow[xl + p] = o[p];
                }
                load(u, y + R + D + 1);                     // the slot of row y-R
            }
        }
    }
}

}  // namespace stb200
