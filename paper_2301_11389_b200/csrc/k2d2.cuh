// k2d2.cuh — two (or three) sweeps per HBM pass for the large 2-D ping-pong runs
// ("multiple sweeps per HBM pass"), register-cache
// form of k2d.cuh.
//
// A single sweep of the 2-D kinds is HBM-bound at ~8 B/pt (k2d runs at
// 0.96-1.04 of the copy peak), so the only way past that roofline is to
// read and write each element once per TWO sweeps.  Per warp, per staged
// input row:
//
//   input row -> register window (as k2d: LDS.128 + x halo)
//            -> sweep-1 row (Op::point, the same arithmetic as k2d; cells
//               on the grid's boundary ring keep their input value — the
//               Dirichlet ring stencil_run holds fixed)
//            -> sweep-1 register window (x halo of the sweep-1 row from the
//               neighbour lanes: shfl.up/down for SHUFFLE, a per-warp staged
//               row in shared memory for PLAIN)
//            -> sweep-2 row (Op::point again) -> STG.128.
//
// Overlapped warp tiles: a warp computes sweep 1 on its 32 lanes x V
// columns; lanes 0 and 31 lack one side of the sweep-1 halo, so sweep-2
// results are stored by lanes 1..30 only (30 V columns per warp, 120 fp32).
// Adjacent warps' tiles overlap by 2 V columns (6.7% redundant sweep-1
// work).  A strip of H sweep-2 rows reads H + 4R input rows (the 2R extra
// rows on each side are shared with the neighbouring strips through L2).
// Results are bit-identical to two separate k2d sweeps.
//
// NSW = 3 chains one more level the same way (sweep-2 rows -> sweep-2
// register window -> sweep-3 row); each level loses one lane per side, so
// lanes 2..29 store (28 V columns per warp) and a strip reads H + 6R rows.
#pragma once
#include "k2d.cuh"

namespace stb200 {

#ifndef STB200_2D2_S
#define STB200_2D2_S 16           // staged rows per CTA (ring stages); power of 2
#endif
constexpr int kStages2D2 = STB200_2D2_S;
// STB200_2D2_CT = 1: the ring has a multiple of the window height NW = 2R+1
// stages and the march is unrolled by the stage count, so a row's ring slot,
// its mbarriers and the stage it releases are compile-time constants (only
// the phase bit is carried); 0: power-of-two ring, slots computed per row.
// Measured (profiles/r02_ab_ct.txt, Gpt/s SHUFFLE / PLAIN, power-of-two 16
// stages -> compile-time slots): jacobi2d5 fp32 32768^2 2016 / 1665 -> 2043 /
// 1687, jacobi2d9 1588 / 1536 -> 1636 / 1634, gaussblur 8192^2 x100 1363 /
// 1384 -> 1380 / 1395 (10 stages, PLAIN releases in pairs; 20 stages: SHUFFLE
// 1228, batches of 5: PLAIN 1260), fp64 jacobi2d5 even.
#ifndef STB200_2D2_CT
#define STB200_2D2_CT 1
#endif
#ifndef STB200_2D2_S2
#define STB200_2D2_S2 10          // CT ring stages for radius 2 (a multiple of 5)
#endif
#ifndef STB200_2D2_RBS
#define STB200_2D2_RBS 2          // CT: SHUFFLE release batch (2: gaussblur 1378 -> 1391, Jacobi even)
#endif
#ifndef STB200_2D2_RBP
#define STB200_2D2_RBP 0          // CT: PLAIN release batch (0: 4 if it divides S, else 2)
#endif
// compile-time slots for the 32-bit kernels (the fp64 three-sweep kernels
// would spill at their register cap: 136 / 116 bytes)
template <int R, typename T> constexpr bool k2d2_ct() { return STB200_2D2_CT && sizeof(T) == 4; }
template <int R, typename T> constexpr int k2d2_stages() {
    return k2d2_ct<R, T>() ? (R == 1 ? 12 : STB200_2D2_S2) : kStages2D2;
}
template <int NW> __host__ __device__ constexpr int k2d2_threads() { return (NW + 1) * 32; }
#ifndef STB200_2D2_BACKOFF
#define STB200_2D2_BACKOFF 512    // producer: longest nanosleep between polls of a busy stage
#endif
#ifndef STB200_2D2_FBSEL
#define STB200_2D2_FBSEL 1        // SHUFFLE fallback as one load + selects (0: predicated asm loads)
#endif

template <typename T, int NSW = 2> constexpr int k2d2_txo() { return (32 - 2 * (NSW - 1)) * vlen<T>(); }
template <typename T, int NSW, int NW>
constexpr int k2d2_row_elems() { return NW * k2d2_txo<T, NSW>() + 2 * NSW * vlen<T>(); }
template <typename T, int NSW, int NW, int S = kStages2D2>
constexpr size_t k2d2_smem_bytes() {
    return (size_t)S * (k2d2_row_elems<T, NSW, NW>() * sizeof(T) + 2 * sizeof(uint64_t)) +
           (size_t)(NSW - 1) * NW * (32 + 2) * vlen<T>() * sizeof(T);   // PLAIN: per-warp, per-level sweep row
}

// Consumer warps per CTA (+1 producer warp) and minimum resident CTAs per
// SM (the register cap of __launch_bounds__), per instance.  Eight consumer
// warps and two CTAs (18 warps, <= 96 registers) where the kernel fits: the
// producer warp's registers are shared by twice the consumers.  Measured on
// B200 (10 steps, Gpt/s SHUFFLE / PLAIN, profiles/r02_ab_minb.txt,
// r02_ab_nw8.txt), against 4 consumer warps at 3 CTAs (the registers' limit):
//   jacobi2d5 fp32 32768^2 three sweeps 1908 / 1627 -> 2019 / 1669,
//   jacobi2d5 fp64 16384^2 three sweeps 914 / 789 -> 987 / 813,
//   jacobi2d9 fp32 two sweeps 1508 / 1537 -> 1610 / 1547 (4 x 4 warps),
//   gaussblur separable fp32 8192^2 two sweeps 1205 / 1353 -> 1361 / 1390.
// The others keep 4 consumer warps and as many CTAs as their registers
// allow.  -DSTB200_2D2_NW / -DSTB200_2D2_MINB override every instance (A/Bs).
template <class Op, typename T, int VAR, int NSW>
constexpr int k2d2_nw() {
#ifdef STB200_2D2_NW
    return STB200_2D2_NW;
#else
    if (std::is_same<Op, OpJacobi2D5<T>>::value || std::is_same<Op, OpJacobi2D9<T>>::value) return 8;
    if (IsSep<Op>::value && sizeof(T) == 4 && NSW == 2) return 8;
    return 4;
#endif
}
template <class Op, typename T, int VAR, int NSW>
constexpr int k2d2_minb() {
#ifdef STB200_2D2_MINB
    return STB200_2D2_MINB;
#else
    return k2d2_nw<Op, T, VAR, NSW>() == 8 ? 2 : 1;
#endif
}

// Grid: x = ceil(nx / (NW * TXO)), y = strips of H output rows
// covering [y_lo, y_hi) (R <= y_lo, y_hi <= ny - R).  NSW sweeps per launch.
template <class Op, typename T, int VARIANT, int NSW = 2>
__global__ void __launch_bounds__(k2d2_threads<k2d2_nw<Op, T, VARIANT, NSW>()>(), (k2d2_minb<Op, T, VARIANT, NSW>()))
k2d2(const T* __restrict__ in, T* __restrict__ out, int64_t nx, int ny, int y_lo, int y_hi, int H,
     Coeffs<T, Op::NC> c) {
    static_assert(NSW == 2 || NSW == 3, "two or three sweeps per launch");
    constexpr int R = Op::R;
    constexpr int V = vlen<T>();
    constexpr int TXO = k2d2_txo<T, NSW>();
    constexpr int kWarps2D2 = k2d2_nw<Op, T, VARIANT, NSW>();
    constexpr int W = V + 2 * R;
    constexpr int NW = 2 * R + 1;
    constexpr int WS = k2d2_row_elems<T, NSW, kWarps2D2>();
    constexpr int S = k2d2_stages<R, T>();
    static_assert(R <= V, "halo wider than the staging pad");
    constexpr bool CT = k2d2_ct<R, T>();
    static_assert(!CT || S % NW == 0, "compile-time slots: S a multiple of the window height");
    static_assert(CT || (S & (S - 1)) == 0, "power-of-two ring");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * WS * sizeof(T));
    uint64_t* empty = full + S;
    T* s1row = reinterpret_cast<T*>(empty + S);            // PLAIN: [NSW-1][kWarps2D2][32V + 2V]

    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    const int64_t X0 = (int64_t)blockIdx.x * (kWarps2D2 * TXO);       // CTA's first output column
    const int ys = y_lo + (int)blockIdx.y * H;
    const int ye = min(ys + H, y_hi);
    if (ys >= ye) return;                                  // CTA-uniform
    const int row0 = ys - NSW * R;                         // first input row of the strip
    const int nrows = ye - ys + 2 * NSW * R;               // input rows [ys-NSW*R, ye+NSW*R)
    const int64_t n_left = (nx - X0 + TXO - 1) / TXO;
    const int active = n_left < kWarps2D2 ? (int)n_left : kWarps2D2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], active * 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kWarps2D2) {                                // ---- producer warp
        if (lane == 0) {
            // staged element e <-> global column X0 - NSW*V + e; clip to [0, nx)
            const int64_t g_lo = X0 - NSW * V > 0 ? X0 - NSW * V : 0;
            const int64_t g_hi0 = X0 + kWarps2D2 * TXO + NSW * V;
            const int64_t g_hi = g_hi0 < nx ? g_hi0 : nx;
            const uint32_t bytes = (uint32_t)((g_hi - g_lo) * (int64_t)sizeof(T));
            T* dst0 = ring + (g_lo - (X0 - NSW * V));
            unsigned s = 0, ph = 0;                        // slot of row r, phase of its (r / S)-th use
            for (int r = 0; r < nrows; ++r, s = s + 1 == S ? (ph ^= 1u, 0u) : s + 1) {
                if (r >= S) mbar_wait_backoff<STB200_2D2_BACKOFF>(&empty[s], ph ^ 1u);
                const int yin = row0 + r;
                if (yin >= 0 && yin < ny) {
                    mbar_arrive_expect_tx(&full[s], bytes);
                    bulk_g2s(dst0 + s * WS, in + (int64_t)yin * nx + g_lo, bytes, &full[s]);
                } else {
                    mbar_arrive(&full[s]);                 // outside the grid: never used
                }
            }
        }
        return;
    }
    if (warp >= active) return;                            // past the row end

    // ---- consumer warps
    const int64_t xs = X0 + (int64_t)warp * TXO - (NSW - 1) * V;   // column of lane 0
    const int64_t xl = xs + lane * V;                      // first column of this lane
    const int lo_e = warp * TXO + V + lane * V;            // staged element of column xl
    const bool lane0 = lane == 0, lane31 = lane == 31;
    T wl[NSW][NW][W];                                      // level 0: input rows; k: sweep-k rows

    Coeffs<T, Op::NC> cr;
#pragma unroll
    for (int t = 0; t < Op::NC; ++t) cr.c[t] = c.c[t];
    // separable kinds (OpGauss5Sep): a window row keeps the row-pass values
    // in its centre slots.  The held value of a boundary-ring cell (EDGE
    // path, below) is the raw input value, re-read from the row ring: the
    // ring keeps HOLD more rows resident for it.  (Keeping the raw values in
    // the window held ~27 more registers live in the whole kernel; re-reading
    // them from global memory stalled the edge warps on every row: -17%.)
    constexpr unsigned HOLD = IsSep<Op>::value ? (NSW - 1) * R : 0;
    static_assert(STB200_REL_LAG || HOLD == 0, "held rows need the lagged release");
    auto sep_row = [&](T* d) {
        if constexpr (IsSep<Op>::value) {
            T hv[V];
            Op::template rowpass<V>(d, hv, cr);
#pragma unroll
            for (int k = 0; k < V; ++k) d[R + k] = hv[k];
        }
    };
    const uint32_t rt_zero = (uint32_t)((uint64_t)nx >> 48);   // 0 at run time, unknown to the compiler
    // rows released per fence (pipe.cuh ring_release_lagged): 4 for PLAIN,
    // 1 for SHUFFLE; with compile-time slots a divisor of S
    constexpr unsigned RB = VARIANT == VAR_PLAIN ? (STB200_2D2_RBP ? STB200_2D2_RBP : S % 4 == 0 ? 4 : 2) : (CT ? STB200_2D2_RBS : 1);
    static_assert(!CT || S % RB == 0, "release batch divides the ring");
    // consume input row r from ring slot s (= r mod S) whose fill phase is par
    auto consume = [&](unsigned r, unsigned s, unsigned par, T* dst) {
        if constexpr (CT) {
            // release rows r-HOLD-RB .. r-HOLD-1 when (r - HOLD) % RB == 0:
            // slots and condition are compile-time (s is), one runtime guard
            if (STB200_REL_LAG && (s + S - HOLD % S) % RB == 0 && r >= HOLD + RB) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
                for (unsigned k = 0; k < RB; ++k)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                                     smem_u32(&empty[(s + 2 * S - HOLD - RB + k) % S]))
                                 : "memory");
            }
        } else if (STB200_REL_LAG) {
            ring_release_lagged<S, RB, HOLD>(empty, r);   // rows before r - HOLD (pipe.cuh)
        }
        mbar_wait(&full[s], par);
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
#if STB200_2D2_FBSEL
            // warp-edge fallback: one load at lane 0's left
            // or lane 31's right halo address, then selects
            T e[R];
            {
                const T* pe = row + (lane0 ? lo_e - R : lo_e + V);
#pragma unroll
                for (int k = 0; k < R; ++k) e[k] = pe[k];
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                dst[k] = lane0 ? e[k] : dst[k];
                dst[R + V + k] = lane31 ? e[k] : dst[R + V + k];
            }
#else
            lds_pred<T, R>(lane0, row + lo_e - R, dst);     // warp-edge fallback
            lds_pred<T, R>(lane31, row + lo_e + V, dst + R + V);
#endif
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
        if (!STB200_REL_LAG) mbar_release(&empty[s], dep & rt_zero);
        sep_row(dst);
    };

    // per-element masks: interior columns (sweep 1 computes, else keeps the
    // input value) and the sweep-2 stores (lanes 1..30, interior only)
    bool xin[V];
#pragma unroll
    for (int p = 0; p < V; ++p) xin[p] = xl + p >= R && xl + p < nx - R;
    const bool own = xl < nx && lane >= NSW - 1 && lane <= 32 - NSW;   // lanes whose last sweep is valid
    const bool vec_store = own && xl >= R && xl + V <= nx - R;
    bool el_store[V];
#pragma unroll
    for (int p = 0; p < V; ++p) el_store[p] = !vec_store && own && xin[p];
    // PLAIN staging of sweep level k (1..NSW-1): element e <-> column xs + e.
    // One row per level: with a single row shared by the levels, the
    // three-sweep PLAIN kernel gave run-to-run differences (tools/flake_hunt.py,
    // jacobi2d5 32768^2: 7 of 8 repeats) although __syncwarp orders each reuse.
    auto srow_of = [&](int k) { return s1row + ((k - 1) * kWarps2D2 + warp) * (32 + 2) * V + V; };

    auto point_row = [&](const auto& w, T* o) {
        if constexpr (IsSep<Op>::value && HasPaired<Op>::value) {
#pragma unroll
            for (int p = 0; p < V; p += 2) {
                const float2 r = Op::colpoint2(w, p, cr);
                o[p] = r.x;
                o[p + 1] = r.y;
            }
        } else if constexpr (IsSep<Op>::value) {
#pragma unroll
            for (int p = 0; p < V; ++p) o[p] = Op::colpoint(w, p, cr);
        } else if constexpr (HasPaired<Op>::value) {
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
    };

    // the x halo of a sweep row from the neighbour lanes
    auto halo = [&](const T* v, T* d, int lev) {
#pragma unroll
        for (int k = 0; k < V; ++k) d[R + k] = v[k];
        if constexpr (VARIANT == VAR_SHUFFLE) {
#pragma unroll
            for (int k = 0; k < R; ++k) d[k] = shfl_up(v[V - R + k], 1);
#pragma unroll
            for (int k = 0; k < R; ++k) d[R + V + k] = shfl_down(v[k], 1);
        } else {
            T* srow = srow_of(lev);
            __syncwarp();                                  // previous row's reads are done
            stg_vec(srow + lane * V, v);                   // STS.128 (generic store to smem)
            __syncwarp();
#pragma unroll
            for (int k = 0; k < R; ++k) d[k] = srow[lane * V - R + k];
#pragma unroll
            for (int k = 0; k < R; ++k) d[R + V + k] = srow[lane * V + V + k];
        }
    };

    const int nt = ye - ys + 2 * (NSW - 1) * R;            // sweep-1 rows
    unsigned par_it = 0;                                   // CT: phase of ring pass t / S
    // one staged input row at step t (phase u = t mod NW, compile time after
    // unrolling).  Sweep-1 row y1 = ys - (NSW-1)R + t; sweep-k row
    // y1 - (k-1)R exists once t >= 2R(k-1).  EDGE = false: the warp's columns
    // and the strip's rows are interior at every level and the storing lanes
    // all store whole vectors (no selects, no element stores); decided once
    // per warp, not per row.
    auto step = [&](int t, int u, auto edge_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        {
            const unsigned r = (unsigned)(t + 2 * R);
            if constexpr (CT) {
                // t = it * S + u: slot (u + 2R) mod S and phase are known per u
                consume(r, (unsigned)((u + 2 * R) % S), (par_it ^ (unsigned)(((u + 2 * R) / S) & 1)),
                        wl[0][(u + 2 * R) % NW]);
            } else {
                consume(r, r % S, (r / S) & 1u, wl[0][(u + 2 * R) % NW]);
            }
        }
        const int y1 = ys - (NSW - 1) * R + t;
#pragma unroll
        for (int k = 1; k <= NSW; ++k) {
            if (k > 1 && t < 2 * R * (k - 1)) break;
            const int yk = y1 - (k - 1) * R;
            // level k-1 window centred on row yk: phase u for the input rows,
            // (u + 1) mod NW for a sweep level (its row yk was made R steps ago)
            const int ph = k == 1 ? u : (u + 1) % NW;
            const Win<T, NW, W, R> w{wl[k - 1], ph};
            T v[V];
            point_row(w, v);
            if (k < NSW) {
                if constexpr (EDGE) {
                    const bool yint = yk >= R && yk < ny - R;
#pragma unroll
                    for (int p = 0; p < V; ++p) {               // boundary ring: held value
                        if (!(yint && xin[p]))
                            v[p] = IsSep<Op>::value ? ring[((unsigned)(yk - row0) % S) * WS + lo_e + p]
                                                    : wl[k - 1][(ph + R) % NW][R + p];
                    }
                }
                halo(v, wl[k][u % NW], k);
                sep_row(wl[k][u % NW]);
            } else {
                T* op = out + (int64_t)yk * nx + xl;
                if constexpr (EDGE) {
                    if (vec_store) stg_vec(op, v);
#pragma unroll
                    for (int p = 0; p < V; ++p)
                        if (el_store[p]) op[p] = v[p];
                } else {
                    if (own) stg_vec(op, v);
                }
            }
        }
    };

#pragma unroll
    for (int r = 0; r < 2 * R; ++r) consume((unsigned)r, (unsigned)r, 0u, wl[0][r]);
    auto march = [&](auto edge_tag) {
        int t = 0;
        constexpr int UN = CT ? S : NW;                    // steps per unrolled body
        for (; t + UN <= nt; t += UN, par_it ^= 1u) {
#pragma unroll
            for (int u = 0; u < UN; ++u) step(t + u, u, edge_tag);
        }
#pragma unroll
        for (int u = 0; u < UN - 1; ++u)
            if (t + u < nt) step(t + u, u, edge_tag);
    };
    bool all_x = true;
#pragma unroll
    for (int p = 0; p < V; ++p) all_x = all_x && xin[p];
    const bool stores_lane = lane >= NSW - 1 && lane <= 32 - NSW;
    const bool rows_inner = ys - (NSW - 1) * R >= R && ye + (NSW - 1) * R <= ny - R;
    const bool interior = __all_sync(FULL, all_x && (vec_store || !stores_lane)) && rows_inner;
#ifdef STB200_2D2_NOEDGE
    march(std::false_type{});                              // experiment: register count of the interior path
#else
    if (interior) march(std::false_type{});
    else march(std::true_type{});
#endif
}

}  // namespace stb200
