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
//    x-tiles of the same strip.
//  * S2 row-tile load: lane 0 of each warp streams the warp's row segment
//    (its 32*V elements plus a 16-byte pad each side) into a per-warp ring of
//    kStages2D shared-memory rows with cp.async.bulk (TMA bulk copy, SASS
//    UBLKCP) completing on one mbarrier per stage; ~kStages2D rows per warp
//    are in flight without holding registers.  Every input element is read
//    from HBM once per strip.
//  * S3 x-neighbour taps: each lane reads its own 16-byte vector (LDS.128)
//    into the register window; the R elements left / right of it:
//      SHUFFLE: shfl.sync.up/down by one lane (N = -1 / +1 in lane units);
//      PLAIN:   loads of the same elements from the staged row (LDS).
//  * S4 corner cases: in SHUFFLE lane 0 / lane 31 take their outer halo from
//    the staged row (the %out_of_range fallback load);
//    lanes past the row end read unused pad (the warp stays full: no
//    %incomplete case) and their stores are masked.  The only divergent
//    branch is the store mask in the two edge tiles of a row.
//  * S5 slow-axis taps: the 2R+1 rows of the y-window live in registers,
//    rotated by unrolling (no register moves).
//  * S6 arithmetic: Op::point on the register window, identical code for
//    both variants (so SHUFFLE == PLAIN bit for bit).
//  * S7 store: STG.128 of interior points; the boundary ring is never
//    written.
#pragma once
#include "common.cuh"
#include "pipe.cuh"

namespace stb200 {

constexpr int kWarps2D = 4;       // x-tiles per CTA (128 threads)
constexpr int kStages2D = 8;      // staged rows per warp (bulk copies in flight)

enum { VAR_SHUFFLE = 0, VAR_PLAIN = 1 };

// Read-only view of the register window for output row y at unroll phase u:
// w(dj, e) = element e (0 .. V+2R-1, centre of output p at e = p+R) of input
// row y+dj.  All indices fold to constants after unrolling.
template <typename T, int NW, int W, int R>
struct Win {
    const T (&a)[NW][W];
    int u;
    __device__ __forceinline__ T operator()(int dj, int e) const { return a[(u + R + dj) % NW][e]; }
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
// Shared memory per warp: kStages2D rows of WS = 32*V + 2*PAD elements, PAD =
// one 16-byte vector, + kStages2D mbarriers.
template <typename T>
constexpr int k2d_row_elems() { return 32 * vlen<T>() + 2 * vlen<T>(); }
template <typename T>
constexpr size_t k2d_smem_bytes() {
    return (size_t)kWarps2D * kStages2D * (k2d_row_elems<T>() * sizeof(T) + sizeof(uint64_t));
}

// Grid: x = ceil(ntiles / kWarps2D), y = strips of H output rows covering
// output rows [y_lo, y_hi) (R <= y_lo, y_hi <= ny - R).
template <class Op, typename T, int VARIANT>
__global__ void __launch_bounds__(kWarps2D * 32)
k2d(const T* __restrict__ in, T* __restrict__ out, int64_t nx, int y_lo, int y_hi, int H,
    Coeffs<T, Op::NC> c) {
    constexpr int R = Op::R;
    constexpr int V = vlen<T>();
    constexpr int PAD = V;                 // 16 bytes of halo room each side
    constexpr int W = V + 2 * R;           // lane window width: halo | vector | halo
    constexpr int NW = 2 * R + 1;          // register y-window
    constexpr int WS = k2d_row_elems<T>();
    constexpr int S = kStages2D;
    static_assert(R <= PAD, "halo wider than the staging pad");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    T* ring = reinterpret_cast<T*>(smem_raw) + (size_t)warp * S * WS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kWarps2D * S * WS * sizeof(T)) +
                     warp * S;

    const int64_t x0 = ((int64_t)blockIdx.x * kWarps2D + warp) * (32 * V);
    if (x0 >= nx) return;                                   // warp-uniform
    const int ys = y_lo + (int)blockIdx.y * H;
    const int ye = min(ys + H, y_hi);
    if (ys >= ye) return;
    const int row0 = ys - R;                               // first input row of the strip
    const int nrows = ye - ys + 2 * R;                     // input rows [ys-R, ye+R)

    // Row segment [x0-PAD, x0+32V+PAD) clipped to [0, nx): 16-byte aligned.
    const int64_t g_lo = x0 - PAD > 0 ? x0 - PAD : 0;
    const int64_t g_hi = x0 + 32 * V + PAD < nx ? x0 + 32 * V + PAD : nx;
    const uint32_t seg_bytes = (uint32_t)((g_hi - g_lo) * (int64_t)sizeof(T));
    const int s_off = (int)(g_lo - (x0 - PAD));            // smem element of g_lo

    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
    }
    __syncwarp();
    auto issue = [&](int r) {                              // lane 0 only
        const int s = r % S;
        mbar_arrive_expect_tx(&bars[s], seg_bytes);
        bulk_g2s(ring + s * WS + s_off, in + (int64_t)(row0 + r) * nx + g_lo, seg_bytes, &bars[s]);
    };
    if (lane == 0) {
        for (int r = 0; r < S && r < nrows; ++r) issue(r);
    }

    const int64_t xl = x0 + lane * V;                      // first column of this lane
    const bool own = xl < nx;
    T win[NW][W];

    // S2..S4: row r of the strip -> register window slot `slot`.
    auto consume = [&](int r, T* dst) {
        const int s = r % S;
        mbar_wait(&bars[s], (uint32_t)(r / S) & 1u);
        const T* row = ring + s * WS + PAD;                // element 0 = column x0
        T v[V];
        {
            using VT = typename VecOf<T>::type;
            const VT t = *reinterpret_cast<const VT*>(row + lane * V);
            if constexpr (V == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
            else { v[0] = t.x; v[1] = t.y; }
        }
#pragma unroll
        for (int k = 0; k < V; ++k) dst[R + k] = v[k];
        if constexpr (VARIANT == VAR_SHUFFLE) {
#pragma unroll
            for (int k = 0; k < R; ++k) dst[k] = shfl_up(v[V - R + k], 1);
#pragma unroll
            for (int k = 0; k < R; ++k) dst[R + V + k] = shfl_down(v[k], 1);
            if (lane == 0) {                                // warp edge: the fallback load
#pragma unroll
                for (int k = 0; k < R; ++k) dst[k] = row[k - R];
            }
            if (lane == 31) {
#pragma unroll
                for (int k = 0; k < R; ++k) dst[R + V + k] = row[32 * V + k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < R; ++k) dst[k] = row[lane * V - R + k];
#pragma unroll
            for (int k = 0; k < R; ++k) dst[R + V + k] = row[lane * V + V + k];
        }
        __syncwarp();                                      // every lane has read stage s
        if (lane == 0 && r + S < nrows) {
            fence_proxy_async_smem();
            issue(r + S);
        }
    };

#pragma unroll
    for (int r = 0; r < 2 * R; ++r) consume(r, win[r]);

    const bool vec_store = own && xl >= R && xl + V <= nx - R;
    for (int y0 = ys; y0 < ye; y0 += NW) {
#pragma unroll
        for (int u = 0; u < NW; ++u) {
            const int y = y0 + u;
            if (y < ye) {                                   // warp-uniform
                consume(y - ys + 2 * R, win[(u + 2 * R) % NW]);
                T o[V];
                const Win<T, NW, W, R> w{win, u};
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
            }
        }
    }
}

}  // namespace stb200
