// kgrad.cuh — gradient (SURVEY §8(a) S1-S7 for the 1-input / 3-output kind,
// DESIGN.md §5.2a): a z-marching register-cache kernel without shared-memory
// staging, sized for occupancy instead of for TMA rings.
//
// Why a separate kernel: gradient reads one array and writes three (16 B/pt
// fp32, 12 of them stores).  The store-heavy 1R3W mix needs many warps per SM
// to keep HBM busy (tools/rwmix.cu: 0.88 of the copy peak at 64 warps/SM,
// 0.75 at 16), and k3d's 16-warp / 128-register TMA design is capped at 16.
// Here a warp owns one x-tile (32 lanes x one 16-byte vector) of one row j
// and marches z over a chunk of planes:
//   z taps    a register queue of the centre vectors of planes k-1, k, k+1
//             (each centre vector read from HBM once per chunk);
//   y taps    16-byte loads of rows j-1 / j+1 of plane k — the centre rows of
//             the sibling warps of the same CTA (rows j0..j0+7), so they hit
//             L1 / L2 (ld.global.nc), not HBM;
//   x taps    SHUFFLE: shfl.up / shfl.down of the neighbour lanes' edge
//             elements, one scalar load at the warp edge (§5.1
//             A(tid+N) = B(tid), with the corner-lane fallback load of §5.2);
//             PLAIN: the two neighbour elements re-loaded by every lane (the
//             ORIGINAL code's redundant loads, served by L1).
// Formula (R10, oracle/oracle.c gradient): (ax*(u[i+1]-u[i-1]),
// ay*(u[j+1]-u[j-1]), az*(u[k+1]-u[k-1])), the same expression as k3d's
// OpGradient, so both kernels give identical bits.
#pragma once
#include "common.cuh"

namespace stb200 {

#ifndef STB200_GRAD_WARPS
#define STB200_GRAD_WARPS 8
#endif
constexpr int kGradWarps = STB200_GRAD_WARPS;   // rows per CTA (one warp each)

// Build-time knobs (build.build_experiment A/Bs):
// minimum resident CTAs per SM (register cap 65536 / (256 * MINB)) and
// st.global.cs (evict-first) output stores.
#ifndef STB200_GRAD_MINB
#define STB200_GRAD_MINB (32 / STB200_GRAD_WARPS)
#endif
#ifndef STB200_GRAD_CS
#define STB200_GRAD_CS 0
#endif

template <typename T>
struct GradArgs {
    const T* u;
    T* out[3];
    int64_t nx, ny;
    int z_lo, nzo;        // output planes [z_lo, z_lo + nzo)
    int zc;               // planes per z chunk (blockIdx.z)
    T c[3];
};

template <typename T, int VARIANT>
__global__ void __launch_bounds__(kGradWarps * 32, STB200_GRAD_MINB) kgrad(const __grid_constant__ GradArgs<T> a) {
    constexpr int V = VecOf<T>::V, TX = 32 * V;
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int64_t nx = a.nx, ny = a.ny, sz = nx * ny;
    const int64_t j = 1 + (int64_t)blockIdx.y * kGradWarps + warp;
    if (j > ny - 2) return;                                // whole warp: no block sync below
    const int zb = a.z_lo + (int)blockIdx.z * a.zc;
    const int ze = min(zb + a.zc, a.z_lo + a.nzo);
    if (zb >= ze) return;
    const int64_t i0 = (int64_t)blockIdx.x * TX + (int64_t)lane * V;
    const bool act = i0 < nx;                              // nx % V == 0: whole vector in bounds
    const T* p = a.u + j * nx + (act ? i0 : 0);            // inactive lanes read a valid vector
    const bool has_l = act && i0 > 0, has_r = act && i0 + V < nx;
    const bool full = i0 >= 1 && i0 + V <= nx - 1;         // all V points interior in x
    const int64_t orow = j * nx + i0;

    T cm[V], c0[V], cp[V], yl[V], yh[V];
    T xl = T(0), xr = T(0);
    ldg_vec(cm, p + (int64_t)(zb - 1) * sz);
    ldg_vec(c0, p + (int64_t)zb * sz);
    // software prefetch of plane zb's remaining inputs
    {
        const T* q = p + (int64_t)zb * sz;
        ldg_vec(cp, q + sz);
        ldg_vec(yl, q - nx);
        ldg_vec(yh, q + nx);
        if (VARIANT == 1) {
            if (has_l) xl = __ldg(q - 1);
            if (has_r) xr = __ldg(q + V);
        } else {
            if (lane == 0 && has_l) xl = __ldg(q - 1);
            if (lane == 31 && has_r) xr = __ldg(q + V);
        }
    }
    for (int k = zb; k < ze; ++k) {
        // next plane's loads first (independent of this plane's math)
        T np_[V], nyl[V], nyh[V];
        T nxl = T(0), nxr = T(0);
        const bool more = k + 1 < ze;
        if (more) {
            const T* q = p + (int64_t)(k + 1) * sz;
            ldg_vec(np_, q + sz);
            ldg_vec(nyl, q - nx);
            ldg_vec(nyh, q + nx);
            if (VARIANT == 1) {
                if (has_l) nxl = __ldg(q - 1);
                if (has_r) nxr = __ldg(q + V);
            } else {
                if (lane == 0 && has_l) nxl = __ldg(q - 1);
                if (lane == 31 && has_r) nxr = __ldg(q + V);
            }
        }
        // x taps of this plane
        T left = xl, right = xr;
        if (VARIANT == 0) {
            const T up = shfl_up(c0[V - 1], 1), dn = shfl_down(c0[0], 1);
            if (lane != 0) left = up;
            if (lane != 31) right = dn;
        }
        T gx[V], gy[V], gz[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const T xm = e == 0 ? left : c0[e - 1];
            const T xp = e == V - 1 ? right : c0[e + 1];
            gx[e] = a.c[0] * (xp - xm);
            gy[e] = a.c[1] * (yh[e] - yl[e]);
            gz[e] = a.c[2] * (cp[e] - cm[e]);
        }
        const int64_t o = (int64_t)k * sz + orow;
        if (full) {
            if (STB200_GRAD_CS) {
                stcs_vec(a.out[0] + o, gx);
                stcs_vec(a.out[1] + o, gy);
                stcs_vec(a.out[2] + o, gz);
            } else {
                stg_vec(a.out[0] + o, gx);
                stg_vec(a.out[1] + o, gy);
                stg_vec(a.out[2] + o, gz);
            }
        } else if (act) {
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const int64_t i = i0 + e;
                if (i >= 1 && i <= nx - 2) {
                    a.out[0][o + e] = gx[e];
                    a.out[1][o + e] = gy[e];
                    a.out[2][o + e] = gz[e];
                }
            }
        }
        if (more) {
#pragma unroll
            for (int e = 0; e < V; ++e) {
                cm[e] = c0[e];
                c0[e] = cp[e];
                cp[e] = np_[e];
                yl[e] = nyl[e];
                yh[e] = nyh[e];
            }
            xl = nxl;
            xr = nxr;
        }
    }
}

}  // namespace stb200
