// klap2.cuh — lapgsrb (Table 1; DESIGN.md §3 reading R21) as a
// two-stage staged register-cache kernel: the new red values r are computed
// ONCE per point into a shared-memory plane, and the black outputs read them
// from there (and from the lane's own registers), instead of every black
// output recomputing its six red neighbours from loads.
//
//   r(q)   = interior red q ? w*nb6(u)(q) : u[q]          (stage 1)
//   out(p) = red p ? r(p) : w*(r(p-x)+r(p+x)+r(p-y)+r(p+y)+r(p-z)+r(p+z))   (stage 2)
//
// The same expressions in the same operand order as the oracle (and as the
// first kernel, klapgsrb in kf3.cuh), so results are bit-identical to it.
//
//  * S1 map: CTA = an x-tile of TX = 32*V columns by NR = 32 rows of r
//    (16 consumer warps x 2 rows), i.e. TY = 30 output rows (the r rows
//    above and below are the y halo of stage 2), marching z; LockIter work
//    order (k3d.cuh) on a one-CTA-per-SM persistent grid.
//  * S2 plane load: thread 0 issues one TMA box of u per z-plane:
//    (TX + 2*PADX) columns (one 32-byte sector of the neighbour tiles each
//    side) by NR + 2 rows, zero-filled outside the grid, into an NS-stage ring.
//  * S3 x taps, both stages: SHUFFLE = shfl.up/down of the neighbour lanes'
//    u elements (stage 1) and of the neighbour lanes' r values (stage 2);
//    PLAIN = the neighbour elements read from the staged u box / the r plane.
//  * S4 corner cases: lane 0 / 31 compute r at x0-1 / x0+TX from the staged
//    sectors (one LDS.64 + four LDS whose address is lane 0's or the
//    others'), store it into the r plane's pad, and read it back there in
//    stage 2 (the fallback load of PAPER.md:561-564).
//  * S5 slow axes: u centre rows of planes z-1, z, z+1 in a register queue;
//    a warp's two rows serve each other's y taps from registers, the rows of
//    the sibling warps come from the staged box (u) or the r plane (r).
//    r of planes z-1, z+1 at the lane's own points: a register queue.
//  * S7 store: STG.128 of interior vectors.
//
// Synchronisation: one named barrier per plane.  It orders the r-plane
// writes of plane z (double-buffered) before their stage-2 reads one plane
// later, and once it has passed no warp reads u stage G-3 any more: thread 0
// then issues the TMA load of a later plane into that stage (bar.sync makes
// the reads performed; a proxy fence orders them before the async write).
#pragma once
#include "k3d.cuh"

namespace stb200 {

constexpr int kLapWarps = 16;    // warps per CTA (thread 0 also issues the TMA loads)

template <typename T>
struct LapLayout {
    static constexpr int V = vlen<T>(), TX = 32 * V;
    static constexpr int RY = 2, NR = kLapWarps * RY;      // r rows per tile
    static constexpr int TY = NR - 2;                      // output rows per tile (at most; Lap2Args::ty)
    static constexpr int PADX = 32 / (int)sizeof(T);       // u box x pad (one sector)
    static constexpr int BX = TX + 2 * PADX, BY = NR + 2;  // u box: rows y0-2 .. y0+NR-1
    static constexpr int STAGE = (BX * BY * (int)sizeof(T) + 127) / 128 * 128;
    static constexpr int RPAD = V;                         // r row: one vector of pad each side
    static constexpr int RX = TX + 2 * RPAD;
    static constexpr int RPLANE = NR * RX * (int)sizeof(T);
#ifndef STB200_LAP_NS
    static constexpr int NS = 8;
#else
    static constexpr int NS = STB200_LAP_NS;
#endif
    static constexpr size_t R_OFF = (size_t)NS * STAGE;
    static constexpr size_t BAR_OFF = R_OFF + 2 * (size_t)RPLANE;
    static constexpr size_t SMEM = BAR_OFF + NS * sizeof(uint64_t);
    static_assert(SMEM <= 232448, "klapgsrb2 shared memory over the 227 KB per-CTA limit");
};
constexpr int klap2_threads() { return kLapWarps * 32; }

template <typename T>
struct Lap2Args {
    T* out;
    int64_t nx, ny, nz;
    int z_lo, nzo;          // output planes [z_lo, z_lo + nzo)
    int ntx, nty;
    int ty;                 // output rows per tile (even, <= LapLayout::TY): the u box has ty + 4 rows
    int zsplit, zc, m;      // LockIter
    T w;
};

// The arrival sequence of a CTA (one u plane each): pieces in LockIter
// order, nseg + 4 planes per piece (u planes z_lo+zo-2 .. z_lo+zo+nseg+1);
// the box origin is computed once per piece.
struct ProdIter {
    LockIter it;
    int ntx;
    int bx = 0, by = 0, z = 0, left = 0;
    __device__ __forceinline__ bool next(int TX, int TY, int padx, int z_lo, int& x, int& y, int& zz) {
        if (left == 0) {
            int64_t col;
            int zo, nseg;
            if (!it.next(col, zo, nseg)) return false;
            bx = (int)(col % ntx) * TX - padx;
            by = (int)(col / ntx) * TY - 2;
            z = z_lo + zo - 2;
            left = nseg + 4;
        }
        x = bx;
        y = by;
        zz = z++;
        --left;
        return true;
    }
};

__device__ __forceinline__ void lap_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(kLapWarps * 32) : "memory");
}

template <typename T, int VARIANT>
__global__ void __launch_bounds__(klap2_threads(), 1)
klapgsrb2(const __grid_constant__ TmapPack<1> tm, const __grid_constant__ Lap2Args<T> a) {
    using L = LapLayout<T>;
    constexpr int V = L::V, TX = L::TX, NS = L::NS, RY = L::RY, NR = L::NR;
    const int TY = a.ty;                                   // runtime tile height (dispatch3d.cu picks it)
    const uint32_t box_bytes = (uint32_t)(L::BX * (TY + 4) * sizeof(T));
    constexpr int BX = L::BX, PADX = L::PADX, RX = L::RX, RPAD = L::RPAD;

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
    T* rbuf = reinterpret_cast<T*>(smem + L::R_OFF);
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int64_t ncols = (int64_t)a.ntx * a.nty;

    // Producer = thread 0, inline: arrival A (one u plane) goes to stage
    // A % NS.  Iteration G reads stages G-2 .. G, so once the barrier of
    // iteration G has passed, stage G-3 is free and arrival G + NS - 3 is
    // issued into it.  (No producer warp: 16 warps keep 128 registers per
    // thread, a 17th would cap them at 96.)
    ProdIter pit{LockIter(ncols, a.nzo, a.zsplit, a.zc, a.m, blockIdx.x, gridDim.x), a.ntx};
    auto produce = [&](uint32_t A) {
        int x, y, z;
        if (!pit.next(TX, TY, PADX, a.z_lo, x, y, z)) return;
        const uint32_t s = A % NS;
        mbar_arrive_expect_tx(&full[s], box_bytes);
        tma_load_3d(smem + (size_t)s * L::STAGE, &tm.m[0], x, y, z, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
        prefetch_tmap(&tm.m[0]);
        for (uint32_t A = 0; A < (uint32_t)(NS - 3); ++A) produce(A);
    }
    __syncthreads();

    // ---- consumer warps: r rows rho = 2*warp + rr (grid row y0 - 1 + rho)
    const T w = a.w;
    const bool lane0 = lane == 0;
    const int64_t nx = a.nx, ny = a.ny, nz = a.nz, plane = nx * ny;
    auto stage = [&](uint32_t gg) { return reinterpret_cast<const T*>(smem + (size_t)(gg % NS) * L::STAGE); };
    auto rplane = [&](int64_t z) { return rbuf + (size_t)(z & 1) * (NR * RX); };
    auto lds_vec = [&](const T* p, T* v) {
        using VT = typename VecOf<T>::type;
        const VT t = *reinterpret_cast<const VT*>(p);
        if constexpr (V == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
        else { v[0] = t.x; v[1] = t.y; }
    };

    T uq[RY][3][V];        // u centre vectors, slot = arrival % 3
    T rq[RY][3][V];        // r at the lane's points, slot = arrival % 3
    uint32_t G = 0;        // arrivals consumed (all pieces)

    LockIter it(ncols, a.nzo, a.zsplit, a.zc, a.m, blockIdx.x, gridDim.x);
    int64_t col;
    int zo, nseg;
    while (it.next(col, zo, nseg)) {
        const int tx = (int)(col % a.ntx), ty = (int)(col / a.ntx);
        const int nxi = (int)nx;                           // rows are < 2^31 elements
        const int x0 = tx * TX, xl = x0 + lane * V;
        const int y0 = ty * TY;
        const bool own = xl < nxi;
        const bool x_vec = own && xl >= 1 && xl + V <= nxi - 1;
        // warp-uniform: every element of the tile row is interior in x (all
        // but the grid-edge tiles), so the red updates need no x mask
        const bool xall = __all_sync(FULL, x_vec);
        bool xin[V];
#pragma unroll
        for (int e = 0; e < V; ++e) xin[e] = xl + e >= 1 && xl + e <= nxi - 2;
        // corner point k = lane & 3 of this warp: row rho_k = 2*warp + (k & 1),
        // left (x0-1, k < 2) or right (x0+TX) of the tile; lanes 4..31 repeat
        // lanes 0..3 (same value, same address)
        const int ck = lane & 3, krr = ck & 1, kside = ck >> 1;
        const int xe = kside ? x0 + TX : x0 - 1;
        const bool xe_in = xe >= 1 && xe <= nxi - 2;
        const int xe_odd = kside ? 0 : 1;                  // x0 is even
        const int ce = (warp * RY + krr + 1) * BX + PADX + (kside ? TX : -1);   // in the u box
        const int cre = (warp * RY + krr) * RX + (kside ? RPAD + TX : RPAD - 1); // in the r plane
        // warp-edge fallback column of the SHUFFLE variant (lane 0: x0-1, lane 31: x0+TX)
        const int fb = PADX + (lane0 ? -1 : TX);
        const int frb = lane0 ? RPAD - 1 : RPAD + TX;
        int gy[RY];
        bool yin[RY], out_ok[RY], act[RY][V];
#pragma unroll
        for (int rr = 0; rr < RY; ++rr) {
            const int rho = warp * RY + rr;
            gy[rr] = y0 - 1 + rho;
            yin[rr] = gy[rr] >= 1 && gy[rr] <= (int)ny - 2;
            out_ok[rr] = yin[rr] && rho >= 1 && rho <= TY;
#pragma unroll
            for (int e = 0; e < V; ++e) act[rr][e] = yin[rr] && (xall || xin[e]);
        }
        const int yk = y0 - 1 + warp * RY + krr;
        const bool ck_in = xe_in && yk >= 1 && yk <= (int)ny - 2;   // corner point inside the grid interior (x, y)
        // warp-uniform: both rows interior in y and every element in x (the
        // red updates then need no mask)
        const bool fast = xall && yin[0] && yin[1];
        bool st_fast[RY];
#pragma unroll
        for (int rr = 0; rr < RY; ++rr) st_fast[rr] = xall && out_ok[rr];
        const int Z0 = a.z_lo + zo - 2;                     // u plane of arrival 0
        const int np = nseg + 4;
        T* obase[RY];
#pragma unroll
        for (int rr = 0; rr < RY; ++rr) obase[rr] = a.out + ((int64_t)(Z0 + 2) * ny + gy[rr]) * nx + xl;
        // the two rows of a warp have opposite colours: par0 = colour of row 0
        const int par0 = (gy[0] + Z0) & 1;                  // at u plane Z0

        // One arrival t (u plane Z0 + t): the centre rows into the queue;
        // S1: r at plane zr = Z0 + t - 1 (u planes t-2, t-1, t); S2: output
        // plane zr - 1 (r planes t-2, t-1, t).  U = t % 3 (queue slots).
        // Both stages' operands are gathered first and their arithmetic
        // shares one colour branch (plane zr and zr - 1 have opposite
        // colours), so the two stages interleave.
        auto arrival = [&](int t, auto U, auto S1, auto S2) {
            constexpr int u = decltype(U)::value;
            constexpr bool s1on = decltype(S1)::value, s2on = decltype(S2)::value;
            constexpr int s0 = u, s1 = (u + 2) % 3, s2 = (u + 1) % 3;   // slots of t, t-1, t-2
            mbar_wait(&full[G % NS], (G / NS) & 1u);
            // every warp has finished arrival t-1: the r plane written two
            // planes ago is free again, and u stage G-3 is read by no one
            lap_bar();
            if (threadIdx.x == 0) {
                fence_proxy_async_smem();                  // the reads of stage G-3 before the TMA write
                produce(G + NS - 3);
            }
            const T* sp = stage(G);
            const uint32_t Gc = G++;
            // (warps whose rows lie beyond a shorter tile compute unused rows:
            // skipping them with an early exit measured 12% slower overall)
#pragma unroll
            for (int rr = 0; rr < RY; ++rr)
                lds_vec(sp + (warp * RY + rr + 1) * BX + PADX + lane * V, uq[rr][s0]);
            if constexpr (s1on) {
                const int zr = Z0 + t - 1;
                const bool zin = zr >= 1 && zr <= (int)nz - 2;
                const T* sc = stage(Gc - 1);
                const T* sm = stage(Gc - 2);
                T* rp = rplane(zr);
                {   // the warp's four corner points (both variants: S2 reads them from the r plane)
                    T s = sc[ce - 1] + sc[ce + 1];
                    s = s + sc[ce - BX];
                    s = s + sc[ce + BX];
                    s = s + sm[ce];
                    s = s + sp[ce];
                    const bool red = ((xe_odd + yk + zr) & 1) == 0;
                    rp[cre] = red && ck_in && zin ? w * s : sc[ce];
                }
                // S1 operands: y taps, x halo of u
                T ym[RY][V], yp[RY][V], xm[RY], xp[RY];
#pragma unroll
                for (int rr = 0; rr < RY; ++rr) {
                    const int row = warp * RY + rr + 1;   // box row of the r row
                    const T* c = uq[rr][s1];
                    if (rr == 0) lds_vec(sc + (row - 1) * BX + PADX + lane * V, ym[rr]);
                    else {
#pragma unroll
                        for (int e = 0; e < V; ++e) ym[rr][e] = uq[0][s1][e];
                    }
                    if (rr == RY - 1) lds_vec(sc + (row + 1) * BX + PADX + lane * V, yp[rr]);
                    else {
#pragma unroll
                        for (int e = 0; e < V; ++e) yp[rr][e] = uq[1][s1][e];
                    }
                    if constexpr (VARIANT == 0) {
                        xm[rr] = shfl_up(c[V - 1], 1);
                        xp[rr] = shfl_down(c[0], 1);
                        const T f = sc[row * BX + fb];        // the warp-edge fallback load
                        xm[rr] = lane0 ? f : xm[rr];
                        xp[rr] = lane == 31 ? f : xp[rr];
                    } else {
                        xm[rr] = sc[row * BX + PADX + lane * V - 1];
                        xp[rr] = sc[row * BX + PADX + lane * V + V];
                    }
                }
                // S2 operands: y taps and x halo of r at plane zr - 1
                const T* rc = rplane(zr - 1);              // complete: written before this arrival's barrier
                T qm[RY][V], qp[RY][V], wm[RY], wp[RY];
                if constexpr (s2on) {
#pragma unroll
                    for (int rr = 0; rr < RY; ++rr) {
                        const int rho = warp * RY + rr;
                        const T* c = rq[rr][s1];
                        if (rr == 0) lds_vec(rc + (rho > 0 ? rho - 1 : 0) * RX + RPAD + lane * V, qm[rr]);
                        else {
#pragma unroll
                            for (int e = 0; e < V; ++e) qm[rr][e] = rq[0][s1][e];
                        }
                        if (rr == RY - 1) lds_vec(rc + (rho + 1 < NR ? rho + 1 : rho) * RX + RPAD + lane * V, qp[rr]);
                        else {
#pragma unroll
                            for (int e = 0; e < V; ++e) qp[rr][e] = rq[1][s1][e];
                        }
                        if constexpr (VARIANT == 0) {
                            wm[rr] = shfl_up(c[V - 1], 1);
                            wp[rr] = shfl_down(c[0], 1);
                            const T f = rc[rho * RX + frb];   // corner r (the fallback load)
                            wm[rr] = lane0 ? f : wm[rr];
                            wp[rr] = lane == 31 ? f : wp[rr];
                        } else {
                            wm[rr] = rc[rho * RX + RPAD + lane * V - 1];
                            wp[rr] = rc[rho * RX + RPAD + lane * V + V];
                        }
                    }
                }
                // element e of row rr is red at plane zr iff (e + rr + P) is
                // even, P = colour of row 0 at zr (xl is even; warp-uniform).
                // S1: r = w*nb6(u) at red elements, u elsewhere.  S2 (plane
                // zr - 1, opposite colours): the black outputs are w times
                // the sum of their six new red neighbours, the red ones r.
                T r[RY][V], o[RY][V];
#pragma unroll
                for (int rr = 0; rr < RY; ++rr)
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        r[rr][e] = uq[rr][s1][e];
                        o[rr][e] = rq[rr][s1][e];
                    }
                auto upd = [&](auto P) {
                    constexpr int pz = decltype(P)::value;
#pragma unroll
                    for (int rr = 0; rr < RY; ++rr) {
                        const T* c = uq[rr][s1];
#pragma unroll
                        for (int e = 0; e < V; ++e) {
                            if (((e + rr + pz) & 1) != 0) continue;
                            T s = (e > 0 ? c[e - 1] : xm[rr]) + (e + 1 < V ? c[e + 1] : xp[rr]);
                            s = s + ym[rr][e];
                            s = s + yp[rr][e];
                            s = s + uq[rr][s2][e];
                            s = s + uq[rr][s0][e];
                            r[rr][e] = w * s;
                        }
                    }
                    T ps[RY][V];                           // S2: the first five taps
                    if constexpr (s2on) {
#pragma unroll
                        for (int rr = 0; rr < RY; ++rr) {
                            const T* c = rq[rr][s1];
#pragma unroll
                            for (int e = 0; e < V; ++e) {
                                if (((e + rr + pz) & 1) != 0) continue;   // black at zr - 1
                                T s = (e > 0 ? c[e - 1] : wm[rr]) + (e + 1 < V ? c[e + 1] : wp[rr]);
                                s = s + qm[rr][e];
                                s = s + qp[rr][e];
                                ps[rr][e] = s + rq[rr][s2][e];
                            }
                        }
                    }
                    // outside the interior r = u (rare: grid-edge tiles and planes)
                    if (!(fast && zin)) {
#pragma unroll
                        for (int rr = 0; rr < RY; ++rr)
#pragma unroll
                            for (int e = 0; e < V; ++e) r[rr][e] = zin && act[rr][e] ? r[rr][e] : uq[rr][s1][e];
                    }
                    if constexpr (s2on) {
#pragma unroll
                        for (int rr = 0; rr < RY; ++rr)
#pragma unroll
                            for (int e = 0; e < V; ++e) {
                                if (((e + rr + pz) & 1) != 0) continue;
                                o[rr][e] = w * (ps[rr][e] + r[rr][e]);   // + r at plane zr (red there)
                            }
                    }
                };
                if (((par0 + t - 1) & 1) == 0) upd(std::integral_constant<int, 0>{});
                else upd(std::integral_constant<int, 1>{});
#pragma unroll
                for (int rr = 0; rr < RY; ++rr) {
#pragma unroll
                    for (int e = 0; e < V; ++e) rq[rr][s0][e] = r[rr][e];
                    st_vec_s(rp + (warp * RY + rr) * RX + RPAD + lane * V, r[rr]);
                }
                if constexpr (s2on) {
#pragma unroll
                    for (int rr = 0; rr < RY; ++rr) {
                        T* op = obase[rr];
                        obase[rr] += plane;
                        if (st_fast[rr]) stg_vec(op, o[rr]);
                        else if (out_ok[rr]) {
                            if (x_vec) stg_vec(op, o[rr]);
                            else if (own) {
#pragma unroll
                                for (int e = 0; e < V; ++e)
                                    if (xin[e]) op[e] = o[rr][e];
                            }
                        }
                    }
                }
            }
        };
        using BT = std::true_type;
        using BF = std::false_type;
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        using I2 = std::integral_constant<int, 2>;
        // prologue (np >= 5): queue only, then r only
        arrival(0, I0{}, BF{}, BF{});
        arrival(1, I1{}, BF{}, BF{});
        arrival(2, I2{}, BT{}, BF{});
        arrival(3, I0{}, BT{}, BF{});
        int t = 4;                                         // slots: t % 3 == 1, 2, 0
        for (; t + 3 <= np; t += 3) {
            arrival(t, I1{}, BT{}, BT{});
            arrival(t + 1, I2{}, BT{}, BT{});
            arrival(t + 2, I0{}, BT{}, BT{});
        }
        if (t < np) arrival(t, I1{}, BT{}, BT{});
        if (t + 1 < np) arrival(t + 1, I2{}, BT{}, BT{});
    }
    (void)plane;
}

}  // namespace stb200
