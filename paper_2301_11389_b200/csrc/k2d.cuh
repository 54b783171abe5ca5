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
//  * S2 row-tile load: a producer warp streams the CTA's row segment into a
//    ring of kStages2D shared-memory rows with cp.async.bulk (TMA bulk copy,
//    SASS UBLKCP) completing on mbarriers; kStages2D rows per CTA are in
//    flight without holding registers.  Every input element is read from HBM
//    once per strip.
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
constexpr int kStages2D = 16;     // staged rows per CTA (bulk copies in flight); power of 2

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
    // fp32: two adjacent outputs (p, p+1) per packed FFMA2 (fma.rn.f32x2):
    // the same per-point FMA chain as point(), fewer issue slots.  A tap
    // whose operand pair (w[e], w[e+1]) starts at an even element is one
    // FFMA2 on an aligned register pair; an odd start would need two moves
    // to build the pair, so it is issued as two scalar FFMAs instead.
    static constexpr bool kPaired = std::is_same<T, float>::value;
    template <class Wn>
    __device__ __forceinline__ static float2 point2(const Wn& w, int p, const Coeffs<T, NC>& c) {
        float2 acc = __fmul2_rn(make_float2(c.c[0], c.c[0]), make_float2(w(-2, p), w(-2, p + 1)));
#pragma unroll
        for (int t = 1; t < 25; ++t) {
            const int dj = t / 5 - 2, e = p + t % 5;
            if ((e & 1) == 0) {
                acc = __ffma2_rn(make_float2(c.c[t], c.c[t]), make_float2(w(dj, e), w(dj, e + 1)), acc);
            } else {
                acc.x = fmaf(c.c[t], w(dj, e), acc.x);
                acc.y = fmaf(c.c[t], w(dj, e + 1), acc.y);
            }
        }
        return acc;
    }
};

// gaussblur5x5 with rank-1 weights w[dj][di] = u[dj] * v[di] (the default
// binomial [1,4,6,4,1]^T [1,4,6,4,1] / 256; api.cu factors the 25 weights at
// create).  Coefficients c = (u[0..4], v[0..4]).  The streaming kernels (k2d,
// k2d2) apply a row pass to every staged row once,
//   h[p] = v0 x[p-2] + v1 x[p-1] + ... + v4 x[p+2]      (one FMA chain),
// keep the row-pass values in the register y-window, and finish with a
// column pass  out = u0 h[y-2] + ... + u4 h[y+2]: 10 FMA per point instead of
// 25.  point() evaluates the same two chains from a raw
// window (30 FMA: the tile / register kernels ktb2d, ktb2r), so every kernel
// family gives the same bits.  The result differs from the 25-term oracle
// order by rounding only (DESIGN.md §7 tolerance).
template <typename T> struct OpGauss5Sep {
    static constexpr int R = 2, NC = 10;
    // fp32: two adjacent points per packed FFMA2 (the same per-point chains;
    // an operand pair starting at an odd element would need two moves, so
    // those taps are two scalar FFMAs, as in OpGauss5::point2)
    static constexpr bool kPaired = std::is_same<T, float>::value;
    template <int V>
    __device__ __forceinline__ static void rowpass(const T* x, T* h, const Coeffs<T, NC>& c) {
        if constexpr (kPaired && V % 2 == 0) {
#pragma unroll
            for (int p = 0; p < V; p += 2) {
                float2 a = __fmul2_rn(make_float2(c.c[5], c.c[5]), make_float2(x[p], x[p + 1]));
#pragma unroll
                for (int d = 1; d < 5; ++d) {
                    if (((p + d) & 1) == 0) {
                        a = __ffma2_rn(make_float2(c.c[5 + d], c.c[5 + d]), make_float2(x[p + d], x[p + d + 1]), a);
                    } else {
                        a.x = fmaf(c.c[5 + d], x[p + d], a.x);
                        a.y = fmaf(c.c[5 + d], x[p + d + 1], a.y);
                    }
                }
                h[p] = a.x;
                h[p + 1] = a.y;
            }
        } else {
#pragma unroll
            for (int p = 0; p < V; ++p) {
                T a = c.c[5] * x[p];
#pragma unroll
                for (int d = 1; d < 5; ++d) a = fma(c.c[5 + d], x[p + d], a);
                h[p] = a;
            }
        }
    }
    // column pass over a window of row-pass values (centre slots e = p + R)
    template <class Wn>
    __device__ __forceinline__ static T colpoint(const Wn& w, int p, const Coeffs<T, NC>& c) {
        const int e = p + R;
        T acc = c.c[0] * w(-2, e);
#pragma unroll
        for (int d = 1; d < 5; ++d) acc = fma(c.c[d], w(d - 2, e), acc);
        return acc;
    }
    // points p, p+1 (p even: the centre slots p+R, p+R+1 are an aligned pair)
    template <class Wn>
    __device__ __forceinline__ static float2 colpoint2(const Wn& w, int p, const Coeffs<T, NC>& c) {
        const int e = p + R;
        float2 acc = __fmul2_rn(make_float2(c.c[0], c.c[0]), make_float2(w(-2, e), w(-2, e + 1)));
#pragma unroll
        for (int d = 1; d < 5; ++d)
            acc = __ffma2_rn(make_float2(c.c[d], c.c[d]), make_float2(w(d - 2, e), w(d - 2, e + 1)), acc);
        return acc;
    }
    // the same value from a window of raw rows
    template <class Wn>
    __device__ __forceinline__ static T point(const Wn& w, int p, const Coeffs<T, NC>& c) {
        auto hrow = [&](int dj) {
            T a = c.c[5] * w(dj, p);
#pragma unroll
            for (int d = 1; d < 5; ++d) a = fma(c.c[5 + d], w(dj, p + d), a);
            return a;
        };
        T acc = c.c[0] * hrow(-2);
#pragma unroll
        for (int d = 1; d < 5; ++d) acc = fma(c.c[d], hrow(d - 2), acc);
        return acc;
    }
};
template <class Op, class = void> struct IsSep : std::false_type {};
template <typename T> struct IsSep<OpGauss5Sep<T>> : std::true_type {};

template <class Op, class = void> struct HasPaired : std::false_type {};
template <class Op> struct HasPaired<Op, std::enable_if_t<Op::kPaired>> : std::true_type {};

// gameoflife: Conway B3/S23 on int cells (Table 1, 9 loads)
struct OpLife {
    static constexpr int R = 1, NC = 0;
    template <class Wn>
    __device__ __forceinline__ static int point(const Wn& w, int p, const Coeffs<int, NC>&) {
        const int e = p + R;
        const int n = w(-1, e - 1) + w(-1, e) + w(-1, e + 1) + w(0, e - 1) + w(0, e + 1)
                    + w(1, e - 1) + w(1, e) + w(1, e + 1);
        // B3/S23 without short-circuit evaluation: no branches (the || / &&
        // form compiled to divergent branches with BSSY/BSYNC around them)
        return (int)((n == 3) | ((n == 2) & (w(0, e) == 1)));
    }
};

// ------------------------------------------------------------------ kernel
// CTA = kWarps2D consumer warps (adjacent x-tiles of one strip) + 1 producer
// warp.  The producer's elected lane streams the CTA's row segment (its
// kWarps2D*32*V elements plus a 16-byte pad each side, 2 KiB + 32 B for
// fp32) into a ring of kStages2D shared-memory rows with cp.async.bulk,
// completion on a "full" mbarrier per stage; consumers release a stage on its
// "empty" mbarrier (every consumer lane arrives: no divergent branch).
template <typename T>
constexpr int k2d_row_elems() { return kWarps2D * 32 * vlen<T>() + 2 * vlen<T>(); }
template <typename T>
constexpr size_t k2d_smem_bytes() {
    return (size_t)kStages2D * (k2d_row_elems<T>() * sizeof(T) + 2 * sizeof(uint64_t));
}
constexpr int k2d_threads() { return (kWarps2D + 1) * 32; }

// Grid: x = ceil(ntiles / kWarps2D), y = strips of H output rows covering
// output rows [y_lo, y_hi) (R <= y_lo, y_hi <= ny - R).
template <class Op, typename T, int VARIANT, bool FUSED = false>
__global__ void __launch_bounds__(k2d_threads())
k2d(const T* __restrict__ in, T* __restrict__ out, int64_t nx, int y_lo, int y_hi, int H,
    Coeffs<T, Op::NC> c, PeerOut<T> peer) {
    constexpr int R = Op::R;
    constexpr int V = vlen<T>();
    constexpr int PAD = V;                 // 16 bytes of halo room each side
    constexpr int W = V + 2 * R;           // lane window width: halo | vector | halo
    constexpr int NW = 2 * R + 1;          // register y-window
    constexpr int WS = k2d_row_elems<T>();
    constexpr int S = kStages2D;
    static_assert(R <= PAD, "halo wider than the staging pad");
    static_assert((S & (S - 1)) == 0, "stage count must be a power of two");
    constexpr unsigned LOG2S = S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * WS * sizeof(T));
    uint64_t* empty = full + S;

    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    const int64_t X0 = (int64_t)blockIdx.x * (kWarps2D * 32 * V);   // CTA's first column
    const int ys = y_lo + (int)blockIdx.y * H;
    const int ye = min(ys + H, y_hi);
    if (ys >= ye) return;                                  // CTA-uniform
    const int row0 = ys - R;                               // first input row of the strip
    const int nrows = ye - ys + 2 * R;                     // input rows [ys-R, ye+R)
    const int64_t nt_left = (nx - X0 + 32 * V - 1) / (32 * V);
    const int active = nt_left < kWarps2D ? (int)nt_left : kWarps2D;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], active * 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kWarps2D) {                                // ---- producer warp
        if (lane == 0) {
            // Row segment [X0-PAD, X0+kWarps2D*32V+PAD) clipped to [0, nx).
            const int64_t g_lo = X0 - PAD > 0 ? X0 - PAD : 0;
            const int64_t g_hi0 = X0 + kWarps2D * 32 * V + PAD;
            const int64_t g_hi = g_hi0 < nx ? g_hi0 : nx;
            const uint32_t bytes = (uint32_t)((g_hi - g_lo) * (int64_t)sizeof(T));
            T* dst0 = ring + (g_lo - (X0 - PAD));
            const T* src = in + (int64_t)row0 * nx + g_lo;
            for (unsigned r = 0; r < (unsigned)nrows; ++r, src += nx) {
                const unsigned s = r & (S - 1);
                if (r >= S) mbar_wait_backoff<256>(&empty[s], ((r >> LOG2S) - 1) & 1u);
                mbar_arrive_expect_tx(&full[s], bytes);
                bulk_g2s(dst0 + s * WS, src, bytes, &full[s]);
            }
        }
        return;
    }
    if (warp >= active) return;                            // past the row end

    // ---- consumer warps
    const int64_t x0 = X0 + warp * (32 * V);
    const int64_t xl = x0 + lane * V;                      // first column of this lane
    const bool own = xl < nx;
    const int lo_e = PAD + warp * 32 * V + lane * V;       // smem element of column xl
    T win[NW][W];

    const bool lane0 = lane == 0, lane31 = lane == 31;
    Coeffs<T, Op::NC> cr;                                  // coefficients held in registers
#pragma unroll
    for (int t = 0; t < Op::NC; ++t) cr.c[t] = c.c[t];
    // S2..S4: strip row r -> register window row dst
    const uint32_t rt_zero = (uint32_t)((uint64_t)nx >> 48);   // 0 at run time, unknown to the compiler
    auto consume = [&](unsigned r, T* dst) {
        const unsigned s = r & (S - 1);
        if (STB200_REL_LAG) ring_release_lagged<S, VARIANT == VAR_PLAIN ? 4 : 1>(empty, r);   // rows before r (pipe.cuh)
        mbar_wait(&full[s], (r >> LOG2S) & 1u);
        const T* row = ring + s * WS;
        T v[V];
        {
            using VT = typename VecOf<T>::type;
            const VT t = *reinterpret_cast<const VT*>(row + lo_e);
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
            // warp-edge lanes: the fallback load from the
            // staged row, predicated on %out_of_range (no branch, no select)
            lds_pred<T, R>(lane0, row + lo_e - R, dst);
            lds_pred<T, R>(lane31, row + lo_e + V, dst + R + V);
        } else {
#pragma unroll
            for (int k = 0; k < R; ++k) dst[k] = row[lo_e - R + k];
#pragma unroll
            for (int k = 0; k < R; ++k) dst[R + V + k] = row[lo_e + V + k];
        }
        // release after the loads completed (pipe.cuh mbar_release): one
        // register of every LDS issued above feeds the (zero) dependency
        uint32_t dep = bits32(dst[0]) ^ bits32(dst[R - 1]) ^ bits32(dst[R + V]) ^ bits32(dst[R + V + R - 1]) ^
                       bits32(dst[R]) ^ bits32(dst[R + V - 1]);
        if (!STB200_REL_LAG) mbar_release(&empty[s], dep & rt_zero);                           // this lane is done with stage s
        if constexpr (IsSep<Op>::value) {                  // separable: the row pass, once per row
            T hv[V];
            Op::template rowpass<V>(dst, hv, cr);
#pragma unroll
            for (int k = 0; k < V; ++k) dst[R + k] = hv[k];
        }
    };

    // S7 masks: whole-vector store for lanes fully inside the interior, else
    // per-element stores of the interior columns (edge tiles only).  Warps
    // whose lanes are all interior take a loop without the element stores.
    const bool vec_store = own && xl >= R && xl + V <= nx - R;
    bool el_store[V];
#pragma unroll
    for (int p = 0; p < V; ++p) el_store[p] = !vec_store && own && xl + p >= R && xl + p < nx - R;

#pragma unroll
    for (int r = 0; r < 2 * R; ++r) consume((unsigned)r, win[r]);

    auto sweep = [&](auto edge_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        T* optr = out + (int64_t)ys * nx + xl;             // running output pointer
        auto emit = [&](int u, int yrow) {
            T o[V];
            const Win<T, NW, W, R> w{win, u};
            if constexpr (IsSep<Op>::value && HasPaired<Op>::value) {            // S6, separable, FFMA2
#pragma unroll
                for (int p = 0; p < V; p += 2) {
                    const float2 r = Op::colpoint2(w, p, cr);
                    o[p] = r.x;
                    o[p + 1] = r.y;
                }
            } else if constexpr (IsSep<Op>::value) {                    // S6, separable
#pragma unroll
                for (int p = 0; p < V; ++p) o[p] = Op::colpoint(w, p, cr);
            } else if constexpr (HasPaired<Op>::value) {                // S6
#pragma unroll
                for (int p = 0; p < V; p += 2) {
                    const float2 r = Op::point2(w, p, cr);
                    o[p] = r.x;
                    o[p + 1] = r.y;
                }
            } else {
#pragma unroll
                for (int p = 0; p < V; ++p) o[p] = Op::point(w, p, cr);
            }
            auto store = [&](T* dst) {
                if constexpr (!EDGE) {
                    stg_vec(dst, o);                                    // S7
                } else {
                    if (vec_store) stg_vec(dst, o);
#pragma unroll
                    for (int p = 0; p < V; ++p)
                        if (el_store[p]) dst[p] = o[p];
                }
            };
            store(optr);
            if constexpr (FUSED) {                         // warp-uniform: halo rows to the peers
                if (peer.lo && yrow < peer.lo_end) store(peer.lo + (optr - out) + peer.d_lo);
                if (peer.hi && yrow >= peer.hi_begin) store(peer.hi + (optr - out) + peer.d_hi);
            }
            optr += nx;
        };
        int y = ys;
        for (; y + NW <= ye; y += NW) {                    // full groups: no guards
#pragma unroll
            for (int u = 0; u < NW; ++u) {
                consume((unsigned)(y + u - ys + 2 * R), win[(u + 2 * R) % NW]);
                emit(u, y + u);
            }
        }
#pragma unroll
        for (int u = 0; u < NW - 1; ++u) {                 // remainder (< NW rows)
            if (y + u < ye) {
                consume((unsigned)(y + u - ys + 2 * R), win[(u + 2 * R) % NW]);
                emit(u, y + u);
            }
        }
    };
    if (__all_sync(FULL, vec_store)) sweep(std::false_type{});
    else sweep(std::true_type{});
}

}  // namespace stb200
