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
    static constexpr int TY = NR - 2;                      // output rows per tile
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
    int zsplit, zc, m;      // LockIter
    T w;
};

// The arrival sequence of a CTA (one u plane each): pieces in LockIter
// order, nseg + 4 planes per piece (u planes z_lo+zo-2 .. z_lo+zo+nseg+1).
struct ProdIter {
    LockIter it;
    int64_t col = 0;
    int zo = 0, nseg = 0, t = 0;
    bool live = false;
    __device__ __forceinline__ bool next(int64_t& c, int& zrel) {   // zrel: plane - z_lo
        if (!live || t >= nseg + 4) {
            if (!it.next(col, zo, nseg)) return false;
            live = true;
            t = 0;
        }
        c = col;
        zrel = zo - 2 + t++;
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
    constexpr int V = L::V, TX = L::TX, NS = L::NS, RY = L::RY, TY = L::TY, NR = L::NR;
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
    ProdIter pit{LockIter(ncols, a.nzo, a.zsplit, a.zc, a.m, blockIdx.x, gridDim.x)};
    auto produce = [&](uint32_t A) {
        int64_t pc;
        int pz;
        if (!pit.next(pc, pz)) return;
        const uint32_t s = A % NS;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(L::BX * L::BY * sizeof(T)));
        tma_load_3d(smem + (size_t)s * L::STAGE, &tm.m[0], (int)(pc % a.ntx) * TX - PADX,
                    (int)(pc / a.ntx) * TY - 2, a.z_lo + pz, &full[s]);
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
        const int64_t x0 = (int64_t)tx * TX, xl = x0 + lane * V;
        const int64_t y0 = (int64_t)ty * TY;
        const bool own = xl < nx;
        const bool x_vec = own && xl >= 1 && xl + V <= nx - 1;
        bool xin[V];
#pragma unroll
        for (int e = 0; e < V; ++e) xin[e] = xl + e >= 1 && xl + e <= nx - 2;
        // the lane's corner point (lane 0: x0-1, the others: x0+TX; lane 31's is used)
        const int64_t xe = lane0 ? x0 - 1 : x0 + TX;
        const bool xe_in = xe >= 1 && xe <= nx - 2;
        const int ce = PADX + (lane0 ? -1 : TX);           // its column in the u box
        int64_t gy[RY];
        bool yin[RY], out_ok[RY];
#pragma unroll
        for (int rr = 0; rr < RY; ++rr) {
            const int rho = warp * RY + rr;
            gy[rr] = y0 - 1 + rho;
            yin[rr] = gy[rr] >= 1 && gy[rr] <= ny - 2;
            out_ok[rr] = yin[rr] && rho >= 1 && rho <= TY;
        }
        const int64_t Z0 = (int64_t)a.z_lo + zo - 2;        // u plane of arrival 0
        const int np = nseg + 4;

        // unrolled by 3 so that the queue slots (arrival % 3) are compile-time
        for (int tb = 0; tb < np; tb += 3) {
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int t = tb + u;
            if (t >= np) break;
            mbar_wait(&full[G % NS], (G / NS) & 1u);
            // every warp has finished iteration t-1: the r plane written two
            // planes ago is free again, and u stage G-3 is read by no one
            lap_bar();
            if (threadIdx.x == 0) {
                fence_proxy_async_smem();                  // the reads of stage G-3 before the TMA write
                produce(G + NS - 3);
            }
            const T* sp = stage(G);
            const uint32_t Gc = G++;
            const int s0 = u, s1 = (u + 2) % 3, s2 = (u + 1) % 3;   // slots of t, t-1, t-2 (unrolled: constants)
#pragma unroll
            for (int rr = 0; rr < RY; ++rr)
                lds_vec(sp + (warp * RY + rr + 1) * BX + PADX + lane * V, uq[rr][s0]);
            if (t < 2) continue;

            // ---- stage 1: r at plane zr = Z0 + t - 1 (u planes t-2, t-1, t)
            const int64_t zr = Z0 + t - 1;
            const bool zin = zr >= 1 && zr <= nz - 2;
            const T* sc = stage(Gc - 1);
            const T* sm = stage(Gc - 2);
            T* rp = rplane(zr);
#pragma unroll
            for (int rr = 0; rr < RY; ++rr) {
                const int rho = warp * RY + rr, row = rho + 1;     // box row of the r row
                const T* c = uq[rr][s1];
                T ym[V], yp[V];
                if (rr == 0) lds_vec(sc + (row - 1) * BX + PADX + lane * V, ym);
                else {
#pragma unroll
                    for (int e = 0; e < V; ++e) ym[e] = uq[0][s1][e];
                }
                if (rr == RY - 1) lds_vec(sc + (row + 1) * BX + PADX + lane * V, yp);
                else {
#pragma unroll
                    for (int e = 0; e < V; ++e) yp[e] = uq[1][s1][e];
                }
                T xm, xp;
                if constexpr (VARIANT == 0) {
                    xm = shfl_up(c[V - 1], 1);
                    xp = shfl_down(c[0], 1);
                } else {
                    xm = sc[row * BX + PADX + lane * V - 1];
                    xp = sc[row * BX + PADX + lane * V + V];
                }
                // corner point of the lane (both variants: stage 2 reads it from the r plane)
                T cl, cc, cr;
                {
                    const T* pr = sc + row * BX + PADX + (lane0 ? -2 : TX);
                    T p0, p1;
                    if constexpr (sizeof(T) == 4) {
                        const float2 t2 = *reinterpret_cast<const float2*>(pr);
                        p0 = t2.x; p1 = t2.y;
                    } else {
                        p0 = pr[0]; p1 = pr[1];
                    }
                    cl = lane0 ? p0 : c[V - 1];
                    cc = lane0 ? p1 : p0;
                    cr = lane0 ? c[0] : p1;
                    if constexpr (VARIANT == 0) {                  // the warp-edge fallback loads
                        if (lane0) xm = p1;
                        if (lane == 31) xp = p0;
                    }
                }
                {
                    T s = cl + cr;
                    s = s + sc[(row - 1) * BX + ce];
                    s = s + sc[(row + 1) * BX + ce];
                    s = s + sm[row * BX + ce];
                    s = s + sp[row * BX + ce];
                    const bool red = ((xe + gy[rr] + zr) & 1) == 0;
                    const T re = red && xe_in && yin[rr] && zin ? w * s : cc;
                    if (lane0) rp[rho * RX + RPAD - 1] = re;
                    if (lane == 31) rp[rho * RX + RPAD + TX] = re;
                }
                T r[V];
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    T s = (e > 0 ? c[e - 1] : xm) + (e + 1 < V ? c[e + 1] : xp);
                    s = s + ym[e];
                    s = s + yp[e];
                    s = s + uq[rr][s2][e];
                    s = s + uq[rr][s0][e];
                    const bool red = ((e + gy[rr] + zr) & 1) == 0;     // xl is even
                    r[e] = red && xin[e] && yin[rr] && zin ? w * s : c[e];
                    rq[rr][s0][e] = r[e];
                }
                st_vec_s(rp + rho * RX + RPAD + lane * V, r);
            }
            if (t < 4) continue;

            // ---- stage 2: output plane zo_ = zr - 1 (r planes t-2, t-1, t)
            const int64_t zo_ = zr - 1;
            const T* rc = rplane(zo_);                     // complete: written before this plane's barrier
#pragma unroll
            for (int rr = 0; rr < RY; ++rr) {
                const int rho = warp * RY + rr;
                const T* c = rq[rr][s1];
                T ym[V], yp[V];
                if (rr == 0) lds_vec(rc + (rho > 0 ? rho - 1 : 0) * RX + RPAD + lane * V, ym);
                else {
#pragma unroll
                    for (int e = 0; e < V; ++e) ym[e] = rq[0][s1][e];
                }
                if (rr == RY - 1) lds_vec(rc + (rho + 1 < NR ? rho + 1 : rho) * RX + RPAD + lane * V, yp);
                else {
#pragma unroll
                    for (int e = 0; e < V; ++e) yp[e] = rq[1][s1][e];
                }
                T xm, xp;
                if constexpr (VARIANT == 0) {
                    xm = shfl_up(c[V - 1], 1);
                    xp = shfl_down(c[0], 1);
                    const T pe = rc[rho * RX + (lane0 ? RPAD - 1 : RPAD + TX)];
                    if (lane0) xm = pe;
                    if (lane == 31) xp = pe;
                } else {
                    xm = rc[rho * RX + RPAD + lane * V - 1];
                    xp = rc[rho * RX + RPAD + lane * V + V];
                }
                T o[V];
#pragma unroll
                for (int e = 0; e < V; ++e) {
                    T s = (e > 0 ? c[e - 1] : xm) + (e + 1 < V ? c[e + 1] : xp);
                    s = s + ym[e];
                    s = s + yp[e];
                    s = s + rq[rr][s2][e];
                    s = s + rq[rr][s0][e];
                    const bool red = ((e + gy[rr] + zo_) & 1) == 0;
                    o[e] = red ? c[e] : w * s;
                }
                if (out_ok[rr]) {
                    T* op = a.out + (zo_ * ny + gy[rr]) * nx + xl;
                    if (x_vec) stg_vec(op, o);
                    else if (own) {
#pragma unroll
                        for (int e = 0; e < V; ++e)
                            if (xin[e]) op[e] = o[e];
                    }
                }
            }
        }
        }
    }
    (void)plane;
}

}  // namespace stb200
