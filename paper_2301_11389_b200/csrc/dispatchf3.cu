// dispatchf3.cu — host launchers of the SURVEY §8(f) row-f3 kernels
// (kf3.cuh): uxx1 and lapgsrb (3-D, z-marching warps), whispering (2-D,
// y-marching warps).  tricubic2 is dispatched to the tricubic kernels
// (dispatch3d.cu): the same function up to rounding order (DESIGN.md §3 R19).
#include <cstdlib>

#include "internal.h"
#include "kf3.cuh"

namespace stb200 {

// z chunk of the z-marching kernels: a chunk restarts the register queues
// (2-3 extra plane loads, L2 hits); 16 planes keeps that under ~15% of the
// loads while leaving enough CTAs for small grids
static int f3_zc() {
    static const int env = getenv("STB200_F3_ZC") ? atoi(getenv("STB200_F3_ZC")) : 0;
    return env > 0 ? env : 16;
}

template <typename T, int VAR>
static cudaError_t launch_uxx1(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                               int64_t z_lo, int64_t z_hi) {
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = 2; z_hi = ld[2] - 1; }
    if (z_hi <= z_lo) return cudaSuccess;
    constexpr int TX = 32 * VecOf<T>::V;
    Uxx1Args<T> a{};
    a.u1 = (const T*)in[0];
    a.d1 = (const T*)in[1];
    a.xx = (const T*)in[2];
    a.xy = (const T*)in[3];
    a.xz = (const T*)in[4];
    a.out = (T*)out[0];
    a.nx = ld[0];
    a.ny = ld[1];
    a.z_lo = (int)z_lo;
    a.nzo = (int)(z_hi - z_lo);
    a.zc = f3_zc();
    for (int t = 0; t < 3; ++t) a.c[t] = (T)h->coeffs[t];
    const int64_t nzc = (a.nzo + a.zc - 1) / a.zc;
    const int64_t nyb = (ld[1] - 3 + kF3Warps - 1) / kF3Warps;
    if (nyb > 65535 || nzc > 65535) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)((ld[0] + TX - 1) / TX), (unsigned)nyb, (unsigned)nzc);
    kuxx1<T, VAR><<<grid, kF3Warps * 32, 0, s>>>(a);
    return cudaGetLastError();
}

template <typename T, int VAR>
static cudaError_t launch_lapgsrb(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                                  int64_t z_lo, int64_t z_hi) {
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = 1; z_hi = ld[2] - 1; }
    if (z_hi <= z_lo) return cudaSuccess;
    constexpr int TX = 32 * VecOf<T>::V;
    LapArgs<T> a{};
    a.u = (const T*)in[0];
    a.out = (T*)out[0];
    a.nx = ld[0];
    a.ny = ld[1];
    a.nz = ld[2];
    a.z_lo = (int)z_lo;
    a.nzo = (int)(z_hi - z_lo);
    a.zc = f3_zc();
    a.w = (T)h->coeffs[0];
    const int64_t nzc = (a.nzo + a.zc - 1) / a.zc;
    const int64_t nyb = (ld[1] - 2 + kF3Warps - 1) / kF3Warps;
    if (nyb > 65535 || nzc > 65535) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)((ld[0] + TX - 1) / TX), (unsigned)nyb, (unsigned)nzc);
    klapgsrb<T, VAR><<<grid, kF3Warps * 32, 0, s>>>(a);
    return cudaGetLastError();
}

template <typename T, int VAR>
static cudaError_t launch_whisper(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                                  int64_t y_lo, int64_t y_hi) {
    const int64_t* ld = h->ldims;
    if (y_lo < 0) { y_lo = 1; y_hi = ld[1] - 1; }
    if (y_hi <= y_lo) return cudaSuccess;
    constexpr int TX = 32 * VecOf<T>::V;
    static const int env_h = getenv("STB200_WH_H") ? atoi(getenv("STB200_WH_H")) : 0;
    WhArgs<T> a{};
    for (int t = 0; t < 8; ++t) a.in[t] = (const T*)in[t];
    for (int t = 0; t < 3; ++t) a.out[t] = (T*)out[t];
    a.nx = ld[0];
    a.ny = ld[1];
    a.y_lo = (int)y_lo;
    a.y_hi = (int)y_hi;
    a.H = env_h > 0 ? env_h : 32;
    const int64_t ntiles = (ld[0] + TX - 1) / TX;
    const int64_t nstrips = (y_hi - y_lo + a.H - 1) / a.H;
    if (nstrips > 65535) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)((ntiles + kF3Warps - 1) / kF3Warps), (unsigned)nstrips);
    kwhisper<T, VAR><<<grid, kF3Warps * 32, 0, s>>>(a);
    return cudaGetLastError();
}


cudaError_t dispatch_f3(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s, int64_t a,
                        int64_t b) {
    const bool f64 = h->dtype == ST_F64, plain = h->variant == ST_PLAIN;
    switch (h->k->kind) {
    case ST_UXX1:
        if (f64) return plain ? launch_uxx1<double, 1>(h, in, out, s, a, b) : launch_uxx1<double, 0>(h, in, out, s, a, b);
        return plain ? launch_uxx1<float, 1>(h, in, out, s, a, b) : launch_uxx1<float, 0>(h, in, out, s, a, b);
    case ST_LAPGSRB:
        if (f64) return plain ? launch_lapgsrb<double, 1>(h, in, out, s, a, b) : launch_lapgsrb<double, 0>(h, in, out, s, a, b);
        return plain ? launch_lapgsrb<float, 1>(h, in, out, s, a, b) : launch_lapgsrb<float, 0>(h, in, out, s, a, b);
    case ST_WHISPERING:
        if (f64) return plain ? launch_whisper<double, 1>(h, in, out, s, a, b) : launch_whisper<double, 0>(h, in, out, s, a, b);
        return plain ? launch_whisper<float, 1>(h, in, out, s, a, b) : launch_whisper<float, 0>(h, in, out, s, a, b);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace stb200
