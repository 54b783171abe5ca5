// klife.cuh — gameoflife (Table 1 "gameoflife"; DESIGN.md §3
// R5) two / three sweeps per HBM pass with the cells packed four to a
// register (one byte per cell, SIMD within a register).
//
// Why: the int32 form of k2d2 spends ~21 instructions per cell and sweep
// (8 adds, 3 compares, selects) and is issue-bound at two sweeps per pass
// (SHUFFLE 0.77 of the copy roofline per launch).  A
// lane's four cells (one 16-byte vector) are packed into the bytes of one
// 32-bit word P (byte p = cell x+p, value 0/1); then per row and sweep
//   horizontal sums  h = P + (P << 8 | left cell) + (P >> 8 | right cell << 24)
//                    (two funnel shifts of the neighbour lanes' words + IADD3)
//   neighbourhood    n9 = h[y-1] + h[y] + h[y+1]   (bytes <= 9: no carries)
//   rule (B3/S23)    alive iff n9 == 3, or n9 == 4 and the cell is alive
//                    (n9 counts the cell itself: n = n9 - c; n == 3 or
//                    (n == 2 and c == 1)  <=>  n9 == 3 or (n9 == 4 and c == 1)),
//                    per byte with carry-free zero tests (bytes < 0x80):
//                    z(x) = ~((x ^ k) + 0x7f7f7f7f) & 0x80808080
// so a sweep of four cells costs ~14 instructions.  The word of a sweep row
// is the next level's input row as is (no unpack between sweeps).
//
// The x taps are the neighbour lanes' words: SHUFFLE = shfl.up/down of the
// packed word (the paper's register cache, moving four cells
// per shuffle); PLAIN = the neighbour cells read back from shared memory
// (level 0: the staged input row; sweep levels: a per-warp staged row).  The
// warp-edge fallback at level 0 is the staged neighbour cell.
//
// Domain: Life's states 0 / 1 (inputs.py draws Bernoulli(1/2)).  A cell's
// value enters as its lowest bit (v & 1), so stale or out-of-grid data can
// never carry into a neighbouring byte; for 0/1 grids the results equal the
// oracle's (and the int32 kernels') bit for bit.  Pipeline, strips and tile
// overlap are those of k2d2.cuh (producer warp, cp.async.bulk row ring,
// lanes NSW-1 .. 32-NSW store).
#pragma once
#include "k2d2.cuh"

namespace stb200 {

constexpr int kWarpsLife = 4;   // consumer warps per CTA (+1 producer); 8 measured even (r02_ab_nw8.txt)

__device__ __forceinline__ uint32_t life_pack(const int* v) {
    const uint32_t a = __byte_perm((uint32_t)v[0], (uint32_t)v[1], 0x0040);
    const uint32_t b = __byte_perm((uint32_t)v[2], (uint32_t)v[3], 0x0040);
    return __byte_perm(a, b, 0x5410) & 0x01010101u;
}
// three-cell horizontal sums of the bytes of P; l / r: words whose byte 3 /
// byte 0 is the cell left of byte 0 / right of byte 3
__device__ __forceinline__ uint32_t life_hsum(uint32_t l, uint32_t p, uint32_t r) {
    return p + __funnelshift_l(l, p, 8) + __funnelshift_r(p, r, 8);
}
// B3/S23 on packed neighbourhood sums n9 (cell included) and cells p
__device__ __forceinline__ uint32_t life_rule(uint32_t n9, uint32_t p) {
    const uint32_t a = (n9 ^ 0x03030303u) + 0x7f7f7f7fu;   // bit 7 of a byte: n9 != 3
    const uint32_t b = (n9 ^ 0x04040404u) + 0x7f7f7f7fu;   // bit 7 of a byte: n9 != 4
    return (((~a) & 0x80808080u) | ((~b) & (p << 7))) >> 7;
}

template <int VARIANT, int NSW = 2>
__global__ void __launch_bounds__(k2d2_threads<kWarpsLife>())
k2dlife(const int* __restrict__ in, int* __restrict__ out, int64_t nx, int ny, int y_lo, int y_hi, int H) {
    static_assert(NSW == 2 || NSW == 3, "two or three sweeps per launch");
    constexpr int R = 1, V = 4, NW = 3;
    constexpr int TXO = k2d2_txo<int, NSW>();
    constexpr int WS = k2d2_row_elems<int, NSW, kWarpsLife>();
    constexpr int S = kStages2D2;
    constexpr unsigned LOG2S = S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    int* ring = reinterpret_cast<int*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * WS * sizeof(int));
    uint64_t* empty = full + S;
    uint32_t* s1row = reinterpret_cast<uint32_t*>(empty + S);   // PLAIN: [kWarpsLife][34] words

    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    const int64_t X0 = (int64_t)blockIdx.x * (kWarpsLife * TXO);
    const int ys = y_lo + (int)blockIdx.y * H;
    const int ye = min(ys + H, y_hi);
    if (ys >= ye) return;
    const int row0 = ys - NSW * R;
    const int nrows = ye - ys + 2 * NSW * R;
    const int64_t n_left = (nx - X0 + TXO - 1) / TXO;
    const int active = n_left < kWarpsLife ? (int)n_left : kWarpsLife;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], active * 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kWarpsLife) {                                // ---- producer warp (as k2d2)
        if (lane == 0) {
            const int64_t g_lo = X0 - NSW * V > 0 ? X0 - NSW * V : 0;
            const int64_t g_hi0 = X0 + kWarpsLife * TXO + NSW * V;
            const int64_t g_hi = g_hi0 < nx ? g_hi0 : nx;
            const uint32_t bytes = (uint32_t)((g_hi - g_lo) * (int64_t)sizeof(int));
            int* dst0 = ring + (g_lo - (X0 - NSW * V));
            for (int r = 0; r < nrows; ++r) {
                const unsigned s = (unsigned)r & (S - 1);
                if (r >= S) mbar_wait_backoff<512>(&empty[s], (((unsigned)r >> LOG2S) - 1) & 1u);
                const int yin = row0 + r;
                if (yin >= 0 && yin < ny) {
                    mbar_arrive_expect_tx(&full[s], bytes);
                    bulk_g2s(dst0 + s * WS, in + (int64_t)yin * nx + g_lo, bytes, &full[s]);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
        }
        return;
    }
    if (warp >= active) return;

    // ---- consumer warps
    const int64_t xs = X0 + (int64_t)warp * TXO - (NSW - 1) * V;
    const int64_t xl = xs + lane * V;
    const int lo_e = warp * TXO + V + lane * V;
    const bool lane0 = lane == 0, lane31 = lane == 31;
    // window of each level: packed centre words and their horizontal sums
    uint32_t wp[NSW][NW], wh[NSW][NW];

    const uint32_t rt_zero = (uint32_t)((uint64_t)nx >> 48);
    auto consume = [&](unsigned r, int slot) {
        const unsigned s = r & (S - 1);
        if (STB200_REL_LAG) ring_release_lagged<S, VARIANT == VAR_PLAIN ? 4 : 1>(empty, r);   // rows before r (pipe.cuh)
        mbar_wait(&full[s], (r >> LOG2S) & 1u);
        const int* row = ring + s * WS;
        int v[V];
        {
            const int4 t = *reinterpret_cast<const int4*>(row + lo_e);
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        }
        const uint32_t p = life_pack(v);
        uint32_t l, rr;
        if constexpr (VARIANT == VAR_SHUFFLE) {
            l = __shfl_up_sync(FULL, p, 1);
            rr = __shfl_down_sync(FULL, p, 1);
            // warp-edge fallback: one load at lane 0's left
            // or lane 31's right neighbour cell, then selects
            const uint32_t e = (uint32_t)row[lane0 ? lo_e - 1 : lo_e + V] & 1u;
            l = lane0 ? e << 24 : l;
            rr = lane31 ? e : rr;
        } else {
            l = ((uint32_t)row[lo_e - 1] & 1u) << 24;
            rr = (uint32_t)row[lo_e + V] & 1u;
        }
        wp[0][slot] = p;
        wh[0][slot] = life_hsum(l, p, rr);
        // release after the loads completed (pipe.cuh mbar_release)
        if (!STB200_REL_LAG) mbar_release(&empty[s], (bits32(v[0]) ^ bits32(v[3]) ^ l ^ rr) & rt_zero);
    };

    // interior columns of the lane as a byte mask (EDGE path: ring cells keep their value)
    uint32_t xmask = 0;
#pragma unroll
    for (int p = 0; p < V; ++p)
        if (xl + p >= R && xl + p < nx - R) xmask |= 0xffu << (8 * p);
    const bool own = xl < nx && lane >= NSW - 1 && lane <= 32 - NSW;
    const bool vec_store = own && xl >= R && xl + V <= nx - R;
    bool el_store[V];
#pragma unroll
    for (int p = 0; p < V; ++p) el_store[p] = !vec_store && own && xl + p >= R && xl + p < nx - R;
    uint32_t* srow = s1row + warp * 34 + 1;                // PLAIN staging: word of lane L at srow[L]

    auto step = [&](int t, int u, auto edge_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        consume((unsigned)(t + 2 * R), (u + 2 * R) % NW);
        const int y1 = ys - (NSW - 1) * R + t;
#pragma unroll
        for (int k = 1; k <= NSW; ++k) {
            if (k > 1 && t < 2 * R * (k - 1)) break;
            const int yk = y1 - (k - 1) * R;
            const int ph = k == 1 ? u : (u + 1) % NW;     // slot of row yk-1 in level k-1
            const uint32_t c = wp[k - 1][(ph + 1) % NW];   // the cells of row yk
            const uint32_t n9 = wh[k - 1][ph] + wh[k - 1][(ph + 1) % NW] + wh[k - 1][(ph + 2) % NW];
            uint32_t q = life_rule(n9, c);
            if (k < NSW) {
                if constexpr (EDGE) {                       // boundary ring: held value
                    const bool yint = yk >= R && yk < ny - R;
                    const uint32_t m = yint ? xmask : 0u;
                    q = (q & m) | (c & ~m);
                }
                uint32_t l, rr;
                if constexpr (VARIANT == VAR_SHUFFLE) {
                    l = __shfl_up_sync(FULL, q, 1);
                    rr = __shfl_down_sync(FULL, q, 1);
                } else {
                    __syncwarp();                          // previous row's reads are done
                    srow[lane] = q;
                    __syncwarp();
                    l = srow[lane - 1];
                    rr = srow[lane + 1];
                }
                wp[k][u % NW] = q;
                wh[k][u % NW] = life_hsum(l, q, rr);
            } else {
                int o[V];
#pragma unroll
                for (int p = 0; p < V; ++p) o[p] = (int)__byte_perm(q, 0u, 0x4440 + p);
                int* op = out + (int64_t)yk * nx + xl;
                if constexpr (EDGE) {
                    if (vec_store) stg_vec(op, o);
#pragma unroll
                    for (int p = 0; p < V; ++p)
                        if (el_store[p]) op[p] = o[p];
                } else {
                    if (own) stg_vec(op, o);
                }
            }
        }
    };

#pragma unroll
    for (int r = 0; r < 2 * R; ++r) consume((unsigned)r, r);
    const int nt = ye - ys + 2 * (NSW - 1) * R;
    auto march = [&](auto edge_tag) {
        int t = 0;
        for (; t + NW <= nt; t += NW) {
#pragma unroll
            for (int u = 0; u < NW; ++u) step(t + u, u, edge_tag);
        }
#pragma unroll
        for (int u = 0; u < NW - 1; ++u)
            if (t + u < nt) step(t + u, u, edge_tag);
    };
    const bool all_x = xmask == 0xffffffffu;
    const bool stores_lane = lane >= NSW - 1 && lane <= 32 - NSW;
    const bool rows_inner = ys - (NSW - 1) * R >= R && ye + (NSW - 1) * R <= ny - R;
    const bool interior = __all_sync(FULL, all_x && (vec_store || !stores_lane)) && rows_inner;
    if (interior) march(std::false_type{});
    else march(std::true_type{});
}

}  // namespace stb200
