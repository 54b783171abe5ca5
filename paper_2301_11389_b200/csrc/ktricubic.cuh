// ktricubic.cuh — tricubic interpolation (Table 1 "tricubic ... 48 / 67",
// PAPER.md:607): g = sum_c wz[c] sum_b wy[b] sum_a wx[a] f[k+c-1][j+b-1][i+a-1]
// with per-point cubic Lagrange weights of the offsets X, Y, Z (DESIGN.md §3
// reading R11).  64 taps of f along a 4x4x4 neighbourhood: 16 x-rows of 4
// taps; in the paper's terms each row is one source load plus 3 shuffles
// (48 shuffles / 67 loads).
//
// The stencil is FP32-pipe bound on B200 (~117 FP ops per point against 20
// compulsory bytes), so the kernel is built around packed FFMA2
// (fma.rn.f32x2): two adjacent output points per instruction, per-point
// weights as register pairs.
//
//  * S1/S2: one CTA per SM, kTriWarps consumer warps (one output row each)
//    + 1 producer warp; per z-plane one TMA box of f ((128+16) x (TY+3):
//    one 32-byte sector each side for the x halo, rows j-1..j+2) into an
//    8-stage ring; the offsets X, Y, Z (read once, no neighbours) are
//    LDG.128 loads issued one output plane ahead; lockstep round-robin work
//    order (LockIter).
//  * S3/S4: per f row, each lane holds its 4 points plus 1 element on the
//    left and 2 on the right: SHUFFLE = shfl.up by 1 / shfl.down by 1 (two
//    values), warp-edge lanes read the staged pad sectors; PLAIN = LDS.
//  * S5: the 4 planes k-1..k+2 stay staged in the ring (no register queue:
//    every tap of every plane is used with per-point weights).
//  * S6: weights, then the 16 row sums, 4 column sums and the plane sum, in
//    the oracle's order (a, then b, then c), as FFMA2 on point pairs.
#pragma once
#include "common.cuh"
#include "k3d.cuh"
#include "pipe.cuh"

namespace stb200 {

constexpr int kTriWarps = 15;     // consumer warps (+1 producer = 16 warps, one CTA per SM)

// Two-point arithmetic: packed FFMA2/FMUL2/FADD2 for fp32, DFMA pairs for fp64.
template <typename T> struct P2;
#ifndef STB200_TRI_SCALAR
template <> struct P2<float> {
    using t = float2;
    __device__ static t mk(float a, float b) { return make_float2(a, b); }
    __device__ static t mul(t a, t b) { return __fmul2_rn(a, b); }
    __device__ static t fma(t a, t b, t c) { return __ffma2_rn(a, b, c); }
    __device__ static t add(t a, t b) { return __fadd2_rn(a, b); }
    __device__ static t sub(t a, t b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
};
#else
template <> struct P2<float> {
    using t = float2;
    __device__ static t mk(float a, float b) { return make_float2(a, b); }
    __device__ static t mul(t a, t b) { return make_float2(a.x * b.x, a.y * b.y); }
    __device__ static t fma(t a, t b, t c) { return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y)); }
    __device__ static t add(t a, t b) { return make_float2(a.x + b.x, a.y + b.y); }
    __device__ static t sub(t a, t b) { return make_float2(a.x - b.x, a.y - b.y); }
};
#endif
template <> struct P2<double> {
    using t = double2;
    __device__ static t mk(double a, double b) { return make_double2(a, b); }
    __device__ static t mul(t a, t b) { return make_double2(a.x * b.x, a.y * b.y); }
    __device__ static t fma(t a, t b, t c) { return make_double2(::fma(a.x, b.x, c.x), ::fma(a.y, b.y, c.y)); }
    __device__ static t add(t a, t b) { return make_double2(a.x + b.x, a.y + b.y); }
    __device__ static t sub(t a, t b) { return make_double2(a.x - b.x, a.y - b.y); }
};

template <typename T>
struct TriLayout {
    static constexpr int ES = (int)sizeof(T), V = 16 / ES, TX = 32 * V, TY = kTriWarps, PADX = 32 / ES;
    static constexpr int FBX = TX + 2 * PADX, FBY = TY + 3;     // f box
    static constexpr int F_BYTES = FBX * FBY * ES;
    static constexpr int STAGE = (F_BYTES + 127) / 128 * 128;
    static constexpr int TX_BYTES = F_BYTES;
    static constexpr int NS = 8;                                // 4 planes in use + 4 in flight
    static constexpr size_t SMEM = (size_t)NS * STAGE + 2 * NS * sizeof(uint64_t);
};

template <typename T>
struct TriArgs {
    const T* X;            // per-point offsets: read with LDG.128, one output plane ahead
    const T* Y;
    const T* Z;
    T* out;
    int64_t nx, ny;
    int z_lo, nzo, ntx, nty, zsplit, zc, m;
};

// Cubic Lagrange weights on nodes {-1, 0, 1, 2} for two points at once:
// L0 = -t(t-1)(t-2)/6, L1 = (t+1)(t-1)(t-2)/2, L2 = -(t+1)t(t-2)/2, L3 = (t+1)t(t-1)/6
template <typename T>
__device__ __forceinline__ void lagrange4x2(typename P2<T>::t t, typename P2<T>::t L[4]) {
    using P = P2<T>;
    const auto one = P::mk(1, 1), two = P::mk(2, 2);
    const auto tm1 = P::sub(t, one), tm2 = P::sub(t, two), tp1 = P::add(t, one);
    const auto a = P::mul(t, tm1);                             // t(t-1)
    const auto b = P::mul(tm1, tm2);                           // (t-1)(t-2)
    const auto c = P::mul(tp1, t);                             // (t+1)t
    const T s6 = T(1) / T(6);
    L[0] = P::mul(P::mul(a, tm2), P::mk(-s6, -s6));
    L[1] = P::mul(P::mul(tp1, b), P::mk(T(0.5), T(0.5)));
    L[2] = P::mul(P::mul(c, tm2), P::mk(T(-0.5), T(-0.5)));
    L[3] = P::mul(P::mul(c, tm1), P::mk(s6, s6));
}

template <typename T, int VARIANT>
__global__ void __launch_bounds__((kTriWarps + 1) * 32, 1)
ktricubic(const __grid_constant__ TmapPack<1> tm, const __grid_constant__ TriArgs<T> args) {
    using L = TriLayout<T>;
    using P = P2<T>;
    using T2 = typename P::t;
    constexpr int NS = L::NS, TX = L::TX, TY = L::TY, PADX = L::PADX, V = L::V, NP = V / 2;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * L::STAGE);
    uint64_t* empty = full + NS;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int64_t ncols = (int64_t)args.ntx * args.nty;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTriWarps * 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kTriWarps) {                               // ---- producer warp
        if (lane == 0) {
            prefetch_tmap(&tm.m[0]);
            uint32_t g = 0;
            LockIter it(ncols, args.nzo, args.zsplit, args.zc, args.m, blockIdx.x, gridDim.x);
            int64_t col;
            int zo, nseg;
            while (it.next(col, zo, nseg)) {
                const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
                const int z_first = args.z_lo + zo - 1;
                for (int t = 0; t < nseg + 3; ++t, ++g) {
                    const uint32_t s = g % NS;
                    if (g >= NS) mbar_wait(&empty[s], (g / NS - 1) & 1u);
                    mbar_arrive_expect_tx(&full[s], L::TX_BYTES);
                    tma_load_3d(smem + (size_t)s * L::STAGE, &tm.m[0], tx * TX - PADX, ty * TY - 1,
                                z_first + t, &full[s]);
                }
            }
        }
        return;
    }

    // ---- consumer warps: output row ty*TY + warp
    const bool lane0 = lane == 0, lane31 = lane == 31;
    uint32_t g = 0;
    const int64_t plane = args.nx * args.ny;
    LockIter it(ncols, args.nzo, args.zsplit, args.zc, args.m, blockIdx.x, gridDim.x);
    int64_t col;
    int zo, nseg;
    while (it.next(col, zo, nseg)) {
        const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
        const int64_t xl = (int64_t)tx * TX + lane * V;
        const int64_t y = (int64_t)ty * TY + warp;
        const bool row_ok = y >= 1 && y < args.ny - 2;
        const bool own = xl < args.nx;
        const bool x_vec = row_ok && own && xl >= 1 && xl + V <= args.nx - 2;
        bool x_el[V];
#pragma unroll
        for (int p = 0; p < V; ++p) x_el[p] = row_ok && !x_vec && own && xl + p >= 1 && xl + p < args.nx - 2;
        T* optr = args.out + ((int64_t)(args.z_lo + zo) * args.ny + y) * args.nx + xl;
        auto stage = [&](uint32_t gg) { return smem + (size_t)(gg % NS) * L::STAGE; };
        auto wait = [&](uint32_t gg) { mbar_wait(&full[gg % NS], (gg / NS) & 1u); };
        // releases carry a zero that depends on the stage's loaded values
        // (pipe.cuh mbar_release): the arrive waits for those loads
        const uint32_t rt_zero = (uint32_t)((uint64_t)args.nx >> 48);
        auto release = [&](uint32_t gg, uint32_t dep) { mbar_release(&empty[gg % NS], dep & rt_zero); };
        auto ldv = [&](const T* p, T* v) {
            using VT = typename VecOf<T>::type;
            const VT t = *reinterpret_cast<const VT*>(p);
            if constexpr (V == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
            else { v[0] = t.x; v[1] = t.y; }
        };

        // offsets of the first output plane; later planes are fetched one
        // plane ahead (clamped address past the grid: values unused)
        const int64_t xoff = (y < args.ny ? y : args.ny - 1) * args.nx + (own ? xl : args.nx - V);
        const T* px = args.X + (int64_t)(args.z_lo + zo) * plane + xoff;
        const T* py = args.Y + (int64_t)(args.z_lo + zo) * plane + xoff;
        const T* pz = args.Z + (int64_t)(args.z_lo + zo) * plane + xoff;
        T Xn[V], Yn[V], Zn[V];
        ldg_vec(Xn, px);
        ldg_vec(Yn, py);
        ldg_vec(Zn, pz);
        wait(g);
        wait(g + 1);
        wait(g + 2);
        for (int o = 0; o < nseg; ++o) {
            T X[V], Y[V], Z[V];
#pragma unroll
            for (int p = 0; p < V; ++p) { X[p] = Xn[p]; Y[p] = Yn[p]; Z[p] = Zn[p]; }
            if (o + 1 < nseg) {
                px += plane; py += plane; pz += plane;
                ldg_vec(Xn, px);
                ldg_vec(Yn, py);
                ldg_vec(Zn, pz);
            }
            wait(g + o + 3);
            // weights of the V points from their offsets X, Y, Z
            T2 wx[NP][4], wy[NP][4], wz[NP][4];
            {
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) {
                    lagrange4x2<T>(P::mk(X[2 * pp], X[2 * pp + 1]), wx[pp]);
                    lagrange4x2<T>(P::mk(Y[2 * pp], Y[2 * pp + 1]), wy[pp]);
                    lagrange4x2<T>(P::mk(Z[2 * pp], Z[2 * pp + 1]), wz[pp]);
                }
            }
            T2 sc[NP];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const T* fb = reinterpret_cast<const T*>(stage(g + o + c));
                T2 sb[NP];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const T* row = fb + (warp + b) * L::FBX + PADX;          // element 0 = column x0
                    T w[V + 3];                                  // columns xl-1 .. xl+V+1
                    ldv(row + lane * V, w + 1);
                    if constexpr (VARIANT == 0) {
                        w[0] = shfl_up(w[V], 1);
                        w[V + 1] = shfl_down(w[1], 1);
                        w[V + 2] = shfl_down(w[2], 1);
                        const T l = row[-1], r0 = row[TX], r1 = row[TX + 1];   // warp-edge fallback
                        w[0] = lane0 ? l : w[0];
                        w[V + 1] = lane31 ? r0 : w[V + 1];
                        w[V + 2] = lane31 ? r1 : w[V + 2];
                    } else {
                        w[0] = row[lane * V - 1];
                        w[V + 1] = row[lane * V + V];
                        w[V + 2] = row[lane * V + V + 1];
                    }
#pragma unroll
                    for (int pp = 0; pp < NP; ++pp) {
                        const int p = 2 * pp;
                        // w[1..V] is the LDS.128 register quad, so the operand
                        // pair (w[e], w[e+1]) is register-aligned for odd e:
                        // one packed FMA there, two scalar FMAs for even e
                        // (instead of two moves to build a pair)
                        T2 sa;
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            const int e = p + a;
                            if (e & 1) {
                                sa = a == 0 ? P::mul(wx[pp][0], P::mk(w[e], w[e + 1]))
                                            : P::fma(wx[pp][a], P::mk(w[e], w[e + 1]), sa);
                            } else if (a == 0) {
                                sa.x = wx[pp][0].x * w[e];
                                sa.y = wx[pp][0].y * w[e + 1];
                            } else {
                                sa.x = ::fma(wx[pp][a].x, w[e], sa.x);
                                sa.y = ::fma(wx[pp][a].y, w[e + 1], sa.y);
                            }
                        }
                        sb[pp] = b == 0 ? P::mul(wy[pp][0], sa) : P::fma(wy[pp][b], sa, sb[pp]);
                    }
                }
#pragma unroll
                for (int pp = 0; pp < NP; ++pp)
                    sc[pp] = c == 0 ? P::mul(wz[pp][0], sb[pp]) : P::fma(wz[pp][c], sb[pp], sc[pp]);
            }
            release(g + o, bits32(sc[0].x) ^ bits32(sc[NP - 1].y));
            T ov[V];
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) { ov[2 * pp] = sc[pp].x; ov[2 * pp + 1] = sc[pp].y; }
            if (x_vec) stg_vec(optr, ov);
#pragma unroll
            for (int p = 0; p < V; ++p)
                if (x_el[p]) optr[p] = ov[p];
            optr += plane;
        }
        release(g + nseg, 0u);
        release(g + nseg + 1, 0u);
        release(g + nseg + 2, 0u);
        g += nseg + 3;
    }
}

}  // namespace stb200
