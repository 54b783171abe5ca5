// kf3.cuh — the SURVEY §8(f) row-f3 suite members on sm_100a: uxx1,
// whispering, lapgsrb (tricubic2 runs the tricubic kernels: the same
// function up to rounding order, DESIGN.md §3 R19).  Formulas: DESIGN.md §3
// R20-R22 and oracle/oracle.c.
//
// All three are HBM-bound multi-array stencils (24, 44 and 8 compulsory
// bytes per fp32 point).  They use the occupancy-first register-cache form
// of kgrad: no shared-memory staging; a warp owns one
// x-tile (32 lanes x one 16-byte vector) and marches along the slowest axis
// keeping the rows / planes it will need again in registers; every input
// vector is one coalesced 16-byte ld.global.nc; taps of other rows of the
// same plane are the sibling warps' rows (L1 / L2 hits).  x-neighbour taps:
//   SHUFFLE  shfl.up / shfl.down of the neighbour lanes' elements — or of a
//            value the neighbour lane already computed from them (whispering's
//            H at x-1, lapgsrb's new red value at x-1 / x+V) — with the
//            paper's corner-case fallback: lanes 0 / 31 load (and compute)
//            what lies outside the warp tile;
//   PLAIN    every lane loads its neighbour elements itself and recomputes
//            the neighbour's intermediate value (the original code's
//            redundant loads).
// Both variants evaluate the same expressions on the same inputs, so their
// results are bit-identical (the tests check it).
#pragma once
#include "common.cuh"

namespace stb200 {

constexpr int kF3Warps = 8;        // warps per CTA (rows of one x-tile, or x-tiles of one strip)

template <typename T>
__device__ __forceinline__ T ldg_or0(bool p, const T* q) { return p ? __ldg(q) : T(0); }
// a*b rounded on its own (never contracted into an FMA): an expression
// evaluated at two sites (a lane's own value, and the neighbour's value
// recomputed by PLAIN / a corner lane) must give the same bits at both
__device__ __forceinline__ float mulrn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mulrn(double a, double b) { return __dmul_rn(a, b); }
// the magnetic half step of one cell: hx = dax Hx - dbx dEz, hy = day Hy + dby dEz
template <typename T>
__device__ __forceinline__ T wh_h(T d, T h, T db, T dez, T sign) { return fma(sign * db, dez, mulrn(d, h)); }

// -------------------------------------------------------------------- uxx1
// out = u1 + (dth/d) (c1 s1 + c2 s2),  d = 0.25 (d1 + d1[j-1] + d1[k-1] + d1[j-1][k-1]),
// s1 / s2 the stagger-1 / stagger-3 differences of xx (x), xy (y), xz (z).
// Warp = row j of an x-tile, marching z over a chunk of zc planes; z queue
// of xz (planes k-2 .. k+1) and d1 (rows j, j-1 of plane k-1).
template <typename T>
struct Uxx1Args {
    const T *u1, *d1, *xx, *xy, *xz;
    T* out;
    int64_t nx, ny;
    int z_lo, nzo, zc;
    T c[3];
};

template <typename T, int VARIANT>
__global__ void __launch_bounds__(kF3Warps * 32) kuxx1(const __grid_constant__ Uxx1Args<T> a) {
    constexpr int V = VecOf<T>::V, TX = 32 * V;
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int64_t nx = a.nx, ny = a.ny, sz = nx * ny;
    const int64_t j = 2 + (int64_t)blockIdx.y * kF3Warps + warp;      // interior rows 2 .. ny-2
    if (j > ny - 2) return;
    const int zb = a.z_lo + (int)blockIdx.z * a.zc;
    const int ze = min(zb + a.zc, a.z_lo + a.nzo);
    if (zb >= ze) return;
    const int64_t i0 = (int64_t)blockIdx.x * TX + (int64_t)lane * V;
    const bool act = i0 < nx;
    const int64_t row = j * nx + (act ? i0 : 0);
    const bool has_l = act && i0 >= 2, has_r = act && i0 + V < nx;
    const bool full = i0 >= 2 && i0 + V <= nx - 1;                   // all V points interior in x

    T xzm2[V], xzm1[V], xz0[V], dp[V], dpm[V];
    ldg_vec(xzm2, a.xz + (int64_t)(zb - 2) * sz + row);
    ldg_vec(xzm1, a.xz + (int64_t)(zb - 1) * sz + row);
    ldg_vec(xz0, a.xz + (int64_t)zb * sz + row);
    ldg_vec(dp, a.d1 + (int64_t)(zb - 1) * sz + row);
    ldg_vec(dpm, a.d1 + (int64_t)(zb - 1) * sz + row - nx);
    for (int k = zb; k < ze; ++k) {
        const int64_t pl = (int64_t)k * sz + row;
        T xzp1[V], u[V], dc[V], dcm[V], xx[V], ym2[V], ym1[V], y0[V], yp1[V];
        ldg_vec(xzp1, a.xz + pl + sz);
        ldg_vec(u, a.u1 + pl);
        ldg_vec(dc, a.d1 + pl);
        ldg_vec(dcm, a.d1 + pl - nx);
        ldg_vec(xx, a.xx + pl);
        ldg_vec(ym2, a.xy + pl - 2 * nx);
        ldg_vec(ym1, a.xy + pl - nx);
        ldg_vec(y0, a.xy + pl);
        ldg_vec(yp1, a.xy + pl + nx);
        // x taps of xx: elements x-2, x-1 (left) and x+V (right)
        T l2, l1, r1;
        if (VARIANT == 0) {
            l2 = shfl_up(xx[V - 2], 1);
            l1 = shfl_up(xx[V - 1], 1);
            r1 = shfl_down(xx[0], 1);
            if (lane == 0) { l2 = ldg_or0(has_l, a.xx + pl - 2); l1 = ldg_or0(has_l, a.xx + pl - 1); }
            if (lane == 31) r1 = ldg_or0(has_r, a.xx + pl + V);
        } else {
            l2 = ldg_or0(has_l, a.xx + pl - 2);
            l1 = ldg_or0(has_l, a.xx + pl - 1);
            r1 = ldg_or0(has_r, a.xx + pl + V);
        }
        T o[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const T xm2 = e >= 2 ? xx[e - 2] : e == 1 ? l1 : l2;
            const T xm1 = e >= 1 ? xx[e - 1] : l1;
            const T xp1 = e + 1 < V ? xx[e + 1] : r1;
            const T d = T(0.25) * (((dc[e] + dcm[e]) + dp[e]) + dpm[e]);
            T s1 = xx[e] - xm1;
            s1 = s1 + y0[e];
            s1 = s1 - ym1[e];
            s1 = s1 + xz0[e];
            s1 = s1 - xzm1[e];
            T s2 = xp1 - xm2;
            s2 = s2 + yp1[e];
            s2 = s2 - ym2[e];
            s2 = s2 + xzp1[e];
            s2 = s2 - xzm2[e];
            o[e] = fma(a.c[0] / d, fma(a.c[1], s1, a.c[2] * s2), u[e]);
        }
        if (full) {
            stg_vec(a.out + pl, o);
        } else if (act) {
#pragma unroll
            for (int e = 0; e < V; ++e)
                if (i0 + e >= 2 && i0 + e <= nx - 2) a.out[pl + e] = o[e];
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
            xzm2[e] = xzm1[e];
            xzm1[e] = xz0[e];
            xz0[e] = xzp1[e];
            dp[e] = dc[e];
            dpm[e] = dcm[e];
        }
    }
}

// -------------------------------------------------------------- whispering
// hx(q) = dax Hx - dbx (Ez[q+y] - Ez[q]); hy(q) = day Hy + dby (Ez[q+x] - Ez[q])
// Hx' = hx(p), Hy' = hy(p), Ez' = Ez + cb ((hy(p) - hy(p-x)) - (hx(p) - hx(p-y)))
// Warp = x-tile of a strip of H rows, marching y.  hx(p-y) is the previous
// row's Hx' (kept in registers; the strip's first row computes it); hy(p-x)
// is the left neighbour's Hy': the previous element, or the left lane's last
// element (SHUFFLE) / recomputed from the loads at x-1 (PLAIN and the
// corner lane 0).
template <typename T>
struct WhArgs {
    const T* in[8];        // Hx, Hy, Ez, dax, dbx, day, dby, cb
    T* out[3];             // Hx', Hy', Ez'
    int64_t nx, ny;
    int y_lo, y_hi, H;     // output rows [y_lo, y_hi), strips of H rows
};

template <typename T, int VARIANT>
__global__ void __launch_bounds__(kF3Warps * 32) kwhisper(const __grid_constant__ WhArgs<T> a) {
    constexpr int V = VecOf<T>::V, TX = 32 * V;
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int64_t nx = a.nx;
    const int64_t i0 = ((int64_t)blockIdx.x * kF3Warps + warp) * TX + (int64_t)lane * V;
    if (((int64_t)blockIdx.x * kF3Warps + warp) * TX >= nx) return;  // whole warp outside
    const int64_t ys = a.y_lo + (int64_t)blockIdx.y * a.H;
    const int64_t ye = min(ys + a.H, (int64_t)a.y_hi);
    if (ys >= ye) return;
    const bool act = i0 < nx;
    const int64_t ic = act ? i0 : 0;
    const bool has_l = act && i0 >= 1, has_r = act && i0 + V < nx;
    const bool full = i0 >= 1 && i0 + V <= nx - 1;
    const T *Hx = a.in[0], *Hy = a.in[1], *Ez = a.in[2], *dax = a.in[3], *dbx = a.in[4], *day = a.in[5],
            *dby = a.in[6], *cb = a.in[7];

    // prologue: Ez rows ys-1, ys and hx(row ys-1)
    T ezm[V], ez0[V], hxm[V];
    {
        const int64_t q = (ys - 1) * nx + ic;
        T hxv[V], dav[V], dbv[V];
        ldg_vec(ezm, Ez + q);
        ldg_vec(ez0, Ez + q + nx);
        ldg_vec(hxv, Hx + q);
        ldg_vec(dav, dax + q);
        ldg_vec(dbv, dbx + q);
#pragma unroll
        for (int e = 0; e < V; ++e) hxm[e] = wh_h(dav[e], hxv[e], dbv[e], ez0[e] - ezm[e], T(-1));
    }
    for (int64_t j = ys; j < ye; ++j) {
        const int64_t q = j * nx + ic;
        T ezp[V], hxv[V], dav[V], dbv[V], hyv[V], dyv[V], dyb[V], cbv[V];
        ldg_vec(ezp, Ez + q + nx);
        ldg_vec(hxv, Hx + q);
        ldg_vec(dav, dax + q);
        ldg_vec(dbv, dbx + q);
        ldg_vec(hyv, Hy + q);
        ldg_vec(dyv, day + q);
        ldg_vec(dyb, dby + q);
        ldg_vec(cbv, cb + q);
        // Ez at x+V (right neighbour of the last element)
        T ezr;
        if (VARIANT == 0) {
            ezr = shfl_down(ez0[0], 1);
            if (lane == 31) ezr = ldg_or0(has_r, Ez + q + V);
        } else {
            ezr = ldg_or0(has_r, Ez + q + V);
        }
        T hx[V], hy[V], o[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
            hx[e] = wh_h(dav[e], hxv[e], dbv[e], ezp[e] - ez0[e], T(-1));
            hy[e] = wh_h(dyv[e], hyv[e], dyb[e], (e + 1 < V ? ez0[e + 1] : ezr) - ez0[e], T(1));
        }
        // hy at x-1 (left neighbour of the first element)
        T hyl;
        {
            auto recompute = [&]() {
                const T dy = ldg_or0(has_l, day + q - 1), hyx = ldg_or0(has_l, Hy + q - 1);
                const T db = ldg_or0(has_l, dby + q - 1), el = ldg_or0(has_l, Ez + q - 1);
                return wh_h(dy, hyx, db, ez0[0] - el, T(1));
            };
            if (VARIANT == 0) {
                hyl = shfl_up(hy[V - 1], 1);
                if (lane == 0) hyl = recompute();
            } else {
                hyl = recompute();
            }
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const T hym = e > 0 ? hy[e - 1] : hyl;
            o[e] = fma(cbv[e], (hy[e] - hym) - (hx[e] - hxm[e]), ez0[e]);
        }
        if (full) {
            stg_vec(a.out[0] + q, hx);
            stg_vec(a.out[1] + q, hy);
            stg_vec(a.out[2] + q, o);
        } else if (act) {
#pragma unroll
            for (int e = 0; e < V; ++e)
                if (i0 + e >= 1 && i0 + e <= nx - 2) {
                    a.out[0][q + e] = hx[e];
                    a.out[1][q + e] = hy[e];
                    a.out[2][q + e] = o[e];
                }
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
            hxm[e] = hx[e];
            ezm[e] = ez0[e];
            ez0[e] = ezp[e];
        }
    }
}

// ----------------------------------------------------------------- lapgsrb
// red(p) = (i+j+k) even; r(q) = interior red q ? w nb6(q) : u[q];
// out(p) = red(p) ? r(p) : w (r(p-x) + r(p+x) + r(p-y) + r(p+y) + r(p-z) + r(p+z)).
// Warp = row j of an x-tile, marching z.  Register queues: row j of planes
// k-2..k+2, rows j-1 / j+1 of planes k-1..k+1; rows j+-2 of plane k are
// loaded per plane (sibling rows: L1 / L2).  The parity of an element is
// (e + j + k) & 1 (x0 is a multiple of V), uniform over the warp.
// New red values at this row / plane are computed at this lane's red
// elements; a black element at e = 0 / V-1 takes r(x-1) / r(x+V) from the
// neighbour lane (SHUFFLE) or recomputes it (PLAIN, corner lanes).
template <typename T>
struct LapArgs {
    const T* u;
    T* out;
    int64_t nx, ny, nz;
    int z_lo, nzo, zc;
    T w;
};

template <typename T, int V>
struct LapCtx {
    // u at (row, plane) offsets relative to (j, k)
    T p0[5][V];            // row j, planes k-2 .. k+2
    T pm[3][V], pp[3][V];  // rows j-1 / j+1, planes k-1 .. k+1
    T ym2[V], yp2[V];      // rows j-2 / j+2, plane k
};

template <typename T, int VARIANT>
__global__ void __launch_bounds__(kF3Warps * 32) klapgsrb(const __grid_constant__ LapArgs<T> a) {
    constexpr int V = VecOf<T>::V, TX = 32 * V;
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int64_t nx = a.nx, ny = a.ny, nz = a.nz, sz = nx * ny;
    const int64_t j = 1 + (int64_t)blockIdx.y * kF3Warps + warp;
    if (j > ny - 2) return;
    const int zb = a.z_lo + (int)blockIdx.z * a.zc;
    const int ze = min(zb + a.zc, a.z_lo + a.nzo);
    if (zb >= ze) return;
    const int64_t i0 = (int64_t)blockIdx.x * TX + (int64_t)lane * V;
    const bool act = i0 < nx;
    const int64_t ic = act ? i0 : 0;
    const bool full = i0 >= 1 && i0 + V <= nx - 1;
    const T w = a.w;
    const T* U = a.u;
    // clamped plane / row indices: out-of-grid taps only feed the r of
    // boundary points (r = u) or non-interior outputs (never stored)
    auto zc_ = [&](int64_t z) { return z < 0 ? (int64_t)0 : z >= nz ? nz - 1 : z; };
    auto yc_ = [&](int64_t y) { return y < 0 ? (int64_t)0 : y >= ny ? ny - 1 : y; };
    auto ld = [&](T* v, int64_t z, int64_t y) { ldg_vec(v, U + (zc_(z) * ny + yc_(y)) * nx + ic); };
    auto at = [&](int64_t z, int64_t y, int64_t x) -> T {   // scalar tap, clamped into the grid
        const int64_t xx = x < 0 ? 0 : x >= nx ? nx - 1 : x;
        return __ldg(U + (zc_(z) * ny + yc_(y)) * nx + xx);
    };
    auto interior = [&](int64_t z, int64_t y, int64_t x) {
        return x >= 1 && x <= nx - 2 && y >= 1 && y <= ny - 2 && z >= 1 && z <= nz - 2;
    };

    T p0[5][V], pm[3][V], pp[3][V];
    for (int t = 0; t < 4; ++t) ld(p0[t], zb - 2 + t, j);     // planes zb-2 .. zb+1 (zb+2 loaded in the loop)
    for (int t = 0; t < 2; ++t) {                              // planes zb-1, zb
        ld(pm[t], zb - 1 + t, j - 1);
        ld(pp[t], zb - 1 + t, j + 1);
    }
    for (int k = zb; k < ze; ++k) {
        T ym2[V], yp2[V];
        ld(p0[4], k + 2, j);
        ld(pm[2], k + 1, j - 1);
        ld(pp[2], k + 1, j + 1);
        ld(ym2, k, j - 2);
        ld(yp2, k, j + 2);
        const int par = (int)((j + k) & 1);      // element e is red iff ((e + par) & 1) == 0
        // x halos (radius 1) of row j at planes k-1, k, k+1 and rows j+-1 at plane k
        T h0l, h0r, hml, hmr, hpl, hpr, zml, zmr, zpl, zpr;
        if (VARIANT == 0) {
            h0l = shfl_up(p0[2][V - 1], 1); h0r = shfl_down(p0[2][0], 1);
            hml = shfl_up(pm[1][V - 1], 1); hmr = shfl_down(pm[1][0], 1);
            hpl = shfl_up(pp[1][V - 1], 1); hpr = shfl_down(pp[1][0], 1);
            zml = shfl_up(p0[1][V - 1], 1); zmr = shfl_down(p0[1][0], 1);
            zpl = shfl_up(p0[3][V - 1], 1); zpr = shfl_down(p0[3][0], 1);
        }
        if (VARIANT == 1 || lane == 0) {
            h0l = at(k, j, i0 - 1); hml = at(k, j - 1, i0 - 1); hpl = at(k, j + 1, i0 - 1);
            zml = at(k - 1, j, i0 - 1); zpl = at(k + 1, j, i0 - 1);
        }
        if (VARIANT == 1 || lane == 31) {
            h0r = at(k, j, i0 + V); hmr = at(k, j - 1, i0 + V); hpr = at(k, j + 1, i0 + V);
            zmr = at(k - 1, j, i0 + V); zpr = at(k + 1, j, i0 + V);
        }
        // new red values: r0 at row j plane k (this lane's elements), rm / rp at
        // rows j-1 / j+1 plane k, rzm / rzp at row j planes k-1 / k+1 (only the
        // elements a black output needs: the same x)
        T r0[V], rm[V], rp[V], rzm[V], rzp[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const int64_t x = i0 + e;
            const bool red = ((e + par) & 1) == 0;
            const T xl0 = e > 0 ? p0[2][e - 1] : h0l, xr0 = e + 1 < V ? p0[2][e + 1] : h0r;
            // row j plane k: red elements
            {
                T s = xl0 + xr0;
                s = s + pm[1][e];
                s = s + pp[1][e];
                s = s + p0[1][e];
                s = s + p0[3][e];
                r0[e] = red && interior(k, j, x) ? w * s : p0[2][e];
            }
            // the neighbours of a black element (red there)
            {
                const T l = e > 0 ? pm[1][e - 1] : hml, r = e + 1 < V ? pm[1][e + 1] : hmr;
                T s = l + r;
                s = s + ym2[e];
                s = s + p0[2][e];
                s = s + pm[0][e];
                s = s + pm[2][e];
                rm[e] = !red && interior(k, j - 1, x) ? w * s : pm[1][e];
            }
            {
                const T l = e > 0 ? pp[1][e - 1] : hpl, r = e + 1 < V ? pp[1][e + 1] : hpr;
                T s = l + r;
                s = s + p0[2][e];
                s = s + yp2[e];
                s = s + pp[0][e];
                s = s + pp[2][e];
                rp[e] = !red && interior(k, j + 1, x) ? w * s : pp[1][e];
            }
            {
                const T l = e > 0 ? p0[1][e - 1] : zml, r = e + 1 < V ? p0[1][e + 1] : zmr;
                T s = l + r;
                s = s + pm[0][e];
                s = s + pp[0][e];
                s = s + p0[0][e];
                s = s + p0[2][e];
                rzm[e] = !red && interior(k - 1, j, x) ? w * s : p0[1][e];
            }
            {
                const T l = e > 0 ? p0[3][e - 1] : zpl, r = e + 1 < V ? p0[3][e + 1] : zpr;
                T s = l + r;
                s = s + pm[2][e];
                s = s + pp[2][e];
                s = s + p0[2][e];
                s = s + p0[4][e];
                rzp[e] = !red && interior(k + 1, j, x) ? w * s : p0[3][e];
            }
        }
        // r at x-1 / x+V (row j, plane k): the neighbour lanes' r0 (SHUFFLE) or
        // recomputed from loads (PLAIN; corner lanes 0 / 31)
        T rl, rr;
        {
            auto r_at = [&](int64_t x) -> T {                          // r at (x, j, k), from loads
                const bool redx = (((x - i0) + par) & 1) == 0;
                const T c = at(k, j, x);
                if (!(redx && interior(k, j, x))) return c;
                T s = at(k, j, x - 1) + at(k, j, x + 1);
                s = s + at(k, j - 1, x);
                s = s + at(k, j + 1, x);
                s = s + at(k - 1, j, x);
                s = s + at(k + 1, j, x);
                return w * s;
            };
            if (VARIANT == 0) {
                rl = shfl_up(r0[V - 1], 1);
                rr = shfl_down(r0[0], 1);
                if (lane == 0) rl = r_at(i0 - 1);
                if (lane == 31) rr = r_at(i0 + V);
            } else {
                rl = r_at(i0 - 1);
                rr = r_at(i0 + V);
            }
        }
        T o[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const bool red = ((e + par) & 1) == 0;
            const T l = e > 0 ? r0[e - 1] : rl, r = e + 1 < V ? r0[e + 1] : rr;
            T s = l + r;
            s = s + rm[e];
            s = s + rp[e];
            s = s + rzm[e];
            s = s + rzp[e];
            o[e] = red ? r0[e] : w * s;
        }
        const int64_t pl = ((int64_t)k * ny + j) * nx + ic;
        if (full) {
            stg_vec(a.out + pl, o);
        } else if (act) {
#pragma unroll
            for (int e = 0; e < V; ++e)
                if (i0 + e >= 1 && i0 + e <= nx - 2) a.out[pl + e] = o[e];
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
#pragma unroll
            for (int t = 0; t < 4; ++t) p0[t][e] = p0[t + 1][e];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                pm[t][e] = pm[t + 1][e];
                pp[t][e] = pp[t + 1][e];
            }
        }
    }
}

}  // namespace stb200
