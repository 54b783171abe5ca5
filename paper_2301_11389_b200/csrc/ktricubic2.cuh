// ktricubic2.cuh — fp32 tricubic interpolation with two output rows per warp
// (the formula of ktricubic.cuh: g = sum_c wz[c] sum_b wy[b] sum_a wx[a]
// f[k+c-1][j+b-1][i+a-1], cubic Lagrange weights of the per-point offsets
// X, Y, Z; DESIGN.md §3 reading R11, Table 1 "tricubic").
//
// Why a second kernel.  At 20 compulsory bytes per point the kind needs
// ~1.1 points/clock/SM to reach the HBM roofline, and the one-row-per-warp
// kernel is bound by the shared-memory/shuffle (MIO) path, not by the FMA
// pipe: every output row reads 16 staged f rows (4 y-taps x 4 planes) plus a
// 3-element x halo per row.  Here each warp owns output rows y and y+1:
//
//  * the 5 f rows y-1..y+3 of a plane serve both rows (10 row reads per
//    output row instead of 16);
//  * the two points (x, y) and (x, y+1) of a lane are one packed pair, so a
//    tap f[r][x+a-1] is a scalar broadcast operand of one FFMA2
//    (`FFMA2 Rd, Rw.F32x2, Rf.F32, Racc`), and the y and z reductions and
//    the weights are FFMA2 on the same pairs — no register moves to build
//    pairs, 84 FMA lane-ops per point for the sums;
//  * the weights cost 8 FFMA2 per axis per pair:
//      h = t(t-1), L0 = h (2-t)/6, L3 = h (t+1)/6, q = 1 - h/2 = -(t-2)(t+1)/2,
//      L2 = q t, L1 = q (1-t)   (the same polynomials as the oracle, refactored);
//  * the warp-edge fallback (lane 0 needs x0-1, lane 31 needs x0+128, x0+129)
//    is one LDS.64 per row whose address is lane 0's or lane 31's, then a
//    select: one wavefront instead of three broadcasts.
//
// Work order: the (column, plane) items are flattened column-major and cut
// into one equal contiguous range per CTA (FlatIter), so every SM gets the
// same number of planes whatever the column count; a range that crosses a
// column restarts the plane pipeline (3 planes).
#pragma once
#include "ktricubic.cuh"

namespace stb200 {

constexpr int kTri2Warps = 11;    // consumer warps (+1 producer = 12 warps: 3 per SMSP, <=168 regs), 2 rows each

#ifndef STB200_TRI2_NS
#define STB200_TRI2_NS 8          // f plane ring stages
#endif
#ifndef STB200_TRI2_NO
#define STB200_TRI2_NO 3          // X/Y/Z offset ring stages
#endif
#ifndef STB200_TRI2_LAG
#define STB200_TRI2_LAG 2         // offsets of output plane o are issued after f plane o + LAG
#endif

struct Tri2Layout {
    static constexpr int V = 4, TX = 128, RY = 2, TY = kTri2Warps * RY, PADX = 8;
    static constexpr int FBX = TX + 2 * PADX, FBY = TY + 3;       // f box: x0-8 .. x0+135, rows y0-1 .. y0+TY+1
    static constexpr int F_BYTES = FBX * FBY * 4;
    static constexpr int STAGE = (F_BYTES + 127) / 128 * 128;
    static constexpr int NS = STB200_TRI2_NS;                    // 4 planes in use + 4 in flight
    // offsets X, Y, Z of one output plane: three (TX x TY) boxes per stage
    static constexpr int O_BYTES = TX * TY * 4;
    static constexpr int OSTAGE = 3 * O_BYTES;
    static constexpr int NO = STB200_TRI2_NO;
    static constexpr size_t SMEM = (size_t)NS * STAGE + (size_t)NO * OSTAGE + 2 * (NS + NO) * sizeof(uint64_t);
};

// Equal contiguous ranges of the column-major (column, plane) sequence.
struct FlatIter {
    int64_t q, qe, nzo;
    __device__ FlatIter(int64_t ncols, int nzo_, unsigned cta, unsigned G) : nzo(nzo_) {
        const int64_t T = ncols * nzo_;
        q = T * cta / G;
        qe = T * (cta + 1) / G;
    }
    __device__ __forceinline__ bool next(int64_t& col, int& zo, int& nseg) {
        if (q >= qe) return false;
        col = q / nzo;
        zo = (int)(q - col * nzo);
        const int64_t e = (col + 1) * nzo < qe ? (col + 1) * nzo : qe;
        nseg = (int)(e - q);
        q = e;
        return true;
    }
};

// Packed fp32 pairs as opaque 64-bit values (inline PTX f32x2 ops): the
// front end cannot split them, so ptxas keeps every pair in an aligned
// register pair and a scalar operand {f, f} becomes the FFMA2 `.F32`
// broadcast form, with no register moves.
using pr = unsigned long long;
__device__ __forceinline__ pr pk(float a, float b) {
    pr r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float plo(pr v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a;
}
__device__ __forceinline__ float phi(pr v) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return b;
}
#ifndef STB200_TRI2_SCALAR
#define STB200_TRI2_SCALAR 0      // experiment: every pair op as two scalar FFMA/FMUL
#endif
#if !STB200_TRI2_SCALAR
__device__ __forceinline__ pr fma2(pr a, pr b, pr c) {
    pr d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ pr mul2(pr a, pr b) {
    pr d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// a * {f, f} (+ c): the tap f is a broadcast operand
__device__ __forceinline__ pr fma2s(pr a, float f, pr c) { return fma2(a, pk(f, f), c); }
__device__ __forceinline__ pr mul2s(pr a, float f) { return mul2(a, pk(f, f)); }
#else
__device__ __forceinline__ pr fma2(pr a, pr b, pr c) {
    return pk(fmaf(plo(a), plo(b), plo(c)), fmaf(phi(a), phi(b), phi(c)));
}
__device__ __forceinline__ pr mul2(pr a, pr b) { return pk(plo(a) * plo(b), phi(a) * phi(b)); }
__device__ __forceinline__ pr fma2s(pr a, float f, pr c) { return pk(fmaf(plo(a), f, plo(c)), fmaf(phi(a), f, phi(c))); }
__device__ __forceinline__ pr mul2s(pr a, float f) { return pk(plo(a) * f, phi(a) * f); }
#endif
__device__ __forceinline__ pr cst(float v) { return pk(v, v); }
__device__ __forceinline__ void ldsv(float* v, const float* p) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}

// Cubic Lagrange weights on nodes {-1,0,1,2} of a point pair from t and
// h = t(t-1):  L0 = h (2-t)/6, L1 = q (1-t), L2 = q t, L3 = h (t+1)/6 with
// q = 1 - h/2 = -(t-2)(t+1)/2 (the oracle's polynomials, refactored).
// Two packed ops per weight (c is a compile-time index after unrolling).
__device__ __forceinline__ pr hpair(pr t) { return mul2(t, fma2(t, cst(1.f), cst(-1.f))); }
__device__ __forceinline__ pr lagrange_one(int c, pr t, pr h) {
    if (c == 0) return mul2(h, fma2(t, cst(-1.f / 6.f), cst(1.f / 3.f)));
    if (c == 3) return mul2(h, fma2(t, cst(1.f / 6.f), cst(1.f / 6.f)));
    const pr q = fma2(h, cst(-0.5f), cst(1.f));
    return c == 2 ? mul2(q, t) : fma2(mul2(q, t), cst(-1.f), q);   // L1 = q - q t
}
// The same four weights of one point, scalar (8 FFMA/FMUL).
__device__ __forceinline__ void lagrange_scalar(float t, float L[4]) {
    const float h = fmaf(t, t, -t);
    const float q = fmaf(h, -0.5f, 1.f);
    L[0] = h * fmaf(t, -1.f / 6.f, 1.f / 3.f);
    L[3] = h * fmaf(t, 1.f / 6.f, 1.f / 6.f);
    L[2] = q * t;
    L[1] = fmaf(-q, t, q);
}

#ifndef STB200_TRI2_RELDEP
#define STB200_TRI2_RELDEP 0
#endif
template <int VARIANT>
__global__ void __launch_bounds__((kTri2Warps + 1) * 32, 1)
ktricubic2(const __grid_constant__ TmapPack<4> tm, const __grid_constant__ TriArgs<float> args) {
    using L = Tri2Layout;
    constexpr int NS = L::NS, TX = L::TX, TY = L::TY, PADX = L::PADX, V = L::V;
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NO = L::NO;
    unsigned char* osm = smem + (size_t)NS * L::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(osm + (size_t)NO * L::OSTAGE);
    uint64_t* empty = full + NS;
    uint64_t* ofull = empty + NS;
    uint64_t* oempty = ofull + NO;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int64_t ncols = (int64_t)args.ntx * args.nty;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTri2Warps * 32);
        }
        for (int s = 0; s < NO; ++s) {
            mbar_init(&ofull[s], 1);
            mbar_init(&oempty[s], kTri2Warps * 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kTri2Warps) {                              // ---- producer warp
        if (lane == 0) {
            for (int a = 0; a < 4; ++a) prefetch_tmap(&tm.m[a]);
            uint32_t g = 0, go = 0;
            FlatIter it(ncols, args.nzo, blockIdx.x, gridDim.x);
            int64_t col;
            int zo, nseg;
            while (it.next(col, zo, nseg)) {
                const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
                const int z_first = args.z_lo + zo - 1;
                for (int t = 0; t < nseg + 3; ++t, ++g) {
                    const uint32_t s = g % NS;
                    if (g >= NS) mbar_wait_backoff<1024>(&empty[s], (g / NS - 1) & 1u);
                    mbar_arrive_expect_tx(&full[s], L::F_BYTES);
                    tma_load_3d(smem + (size_t)s * L::STAGE, &tm.m[0], tx * TX - PADX, ty * TY - 1,
                                z_first + t, &full[s]);
                    // offsets of output plane t-LAG after f plane t
                    const int o = t - STB200_TRI2_LAG;
                    if (o >= 0 && o < nseg) {
                        const uint32_t so = go % NO;
                        if (go >= NO) mbar_wait_backoff<1024>(&oempty[so], (go / NO - 1) & 1u);
                        mbar_arrive_expect_tx(&ofull[so], L::OSTAGE);
                        unsigned char* dst = osm + (size_t)so * L::OSTAGE;
                        for (int a = 0; a < 3; ++a)
                            tma_load_3d(dst + a * L::O_BYTES, &tm.m[1 + a], tx * TX, ty * TY,
                                        args.z_lo + zo + o, &ofull[so]);
                        ++go;
                    }
                }
            }
        }
        return;
    }

    // ---- consumer warps: output rows y0 = ty*TY + 2*warp and y0 + 1
    const bool lane0 = lane == 0, lane31 = lane == 31;
    uint32_t g = 0, go = 0;
    const int64_t plane = args.nx * args.ny;
    FlatIter it(ncols, args.nzo, blockIdx.x, gridDim.x);
    int64_t col;
    int zo, nseg;
    while (it.next(col, zo, nseg)) {
        const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
        const int64_t xl = (int64_t)tx * TX + lane * V;
        const int64_t y0 = (int64_t)ty * TY + 2 * warp;
        const bool own = xl < args.nx;
        bool vec[2], el[2][V];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool row_ok = y0 + h >= 1 && y0 + h < args.ny - 2;
            vec[h] = row_ok && own && xl >= 1 && xl + V <= args.nx - 2;
#pragma unroll
            for (int p = 0; p < V; ++p) el[h][p] = row_ok && !vec[h] && own && xl + p >= 1 && xl + p < args.nx - 2;
        }
        float* optr = args.out + ((int64_t)(args.z_lo + zo) * args.ny + y0) * args.nx + xl;
        auto stage = [&](uint32_t gg) { return reinterpret_cast<const float*>(smem + (size_t)(gg % NS) * L::STAGE); };
        auto wait = [&](uint32_t gg) { mbar_wait(&full[gg % NS], (gg / NS) & 1u); };
        // releases carry a zero that depends on the stage's loaded values
        // (pipe.cuh mbar_release): the arrive waits for those loads
        const uint32_t rt_zero = (uint32_t)((uint64_t)args.nx >> 48);
        auto release = [&](uint32_t gg, uint32_t dep) { mbar_release(&empty[gg % NS], dep & rt_zero); };

        wait(g);
        wait(g + 1);
        wait(g + 2);
        for (int o = 0; o < nseg; ++o, ++go) {
            float Xn[2][V], Yn[2][V], Zn[2][V];
            {
                mbar_wait(&ofull[go % NO], (go / NO) & 1u);
                const float* ob = reinterpret_cast<const float*>(osm + (size_t)(go % NO) * L::OSTAGE) +
                                  2 * warp * TX + lane * V;
                ldsv(Xn[0], ob); ldsv(Xn[1], ob + TX);
                ob += L::O_BYTES / 4;
                ldsv(Yn[0], ob); ldsv(Yn[1], ob + TX);
                ob += L::O_BYTES / 4;
                ldsv(Zn[0], ob); ldsv(Zn[1], ob + TX);
#if STB200_TRI2_RELDEP
                mbar_release(&oempty[go % NO], (bits32(Xn[0][0]) ^ bits32(Xn[1][0]) ^ bits32(Yn[0][0]) ^
                                                bits32(Yn[1][0]) ^ bits32(Zn[0][0]) ^ bits32(Zn[1][0])) & rt_zero);
#else
                mbar_release_fenced(&oempty[go % NO]);
#endif
            }
            // weights of the 4 point pairs (x+p, y0) / (x+p, y0+1).  Row r of a
            // plane (r = 0..4 = y0-1 .. y0+3) enters point y0 with y weight
            // b = r and point y0+1 with b = r-1: the crossed pairs
            // WY[r-1] = (Ly_r(y0), Ly_{r-1}(y0+1)), r = 1..3, and the edge pair
            // WE = (Ly_0(y0), Ly_3(y0+1)) are built from scalar weights so that
            // each pair is a fresh register pair.
            pr wx[V][4], WY[V][3], WE[V], tz[V], hz[V];
#pragma unroll
            for (int p = 0; p < V; ++p) {
                const pr t = pk(Xn[0][p], Xn[1][p]), h = hpair(t);
#pragma unroll
                for (int a = 0; a < 4; ++a) wx[p][a] = lagrange_one(a, t, h);
                float ly0[4], ly1[4];
                lagrange_scalar(Yn[0][p], ly0);
                lagrange_scalar(Yn[1][p], ly1);
#pragma unroll
                for (int r = 1; r <= 3; ++r) WY[p][r - 1] = pk(ly0[r], ly1[r - 1]);
                WE[p] = pk(ly0[0], ly1[3]);
                tz[p] = pk(Zn[0][p], Zn[1][p]);
                hz[p] = hpair(tz[p]);
            }
            wait(g + o + 3);
            pr sc[V];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float* fb = stage(g + o + c);
                pr sb[V];
                float e0[V], e4[V];
#pragma unroll
                for (int r = 0; r < 5; ++r) {
                    const float* row = fb + (2 * warp + r) * L::FBX + PADX;      // element 0 = column x0
                    float w[V + 3];                                              // columns xl-1 .. xl+V+1
                    {
                        const float4 t = *reinterpret_cast<const float4*>(row + lane * V);
                        w[1] = t.x; w[2] = t.y; w[3] = t.z; w[4] = t.w;
                    }
                    if constexpr (VARIANT == 0) {
                        const float up = shfl_up(w[V], 1);
                        const float d1 = shfl_down(w[1], 1), d2 = shfl_down(w[2], 1);
                        // warp-edge fallback: lane 0 reads
                        // (x0-2, x0-1), the others (x0+128, x0+129): one wavefront
                        const float2 e = *reinterpret_cast<const float2*>(row + (lane0 ? -2 : TX));
                        w[0] = lane0 ? e.y : up;
                        w[V + 1] = lane31 ? e.x : d1;
                        w[V + 2] = lane31 ? e.y : d2;
                    } else {
                        w[0] = row[lane * V - 1];
                        const float2 e = *reinterpret_cast<const float2*>(row + lane * V + V);
                        w[V + 1] = e.x;
                        w[V + 2] = e.y;
                    }
#pragma unroll
                    for (int p = 0; p < V; ++p) {
                        if (r == 0) {                       // point y0 only (b = 0)
                            float t = plo(wx[p][0]) * w[p];
#pragma unroll
                            for (int a = 1; a < 4; ++a) t = fmaf(plo(wx[p][a]), w[p + a], t);
                            e0[p] = t;
                        } else if (r == 4) {                // point y0+1 only (b = 3)
                            float t = phi(wx[p][0]) * w[p];
#pragma unroll
                            for (int a = 1; a < 4; ++a) t = fmaf(phi(wx[p][a]), w[p + a], t);
                            e4[p] = t;
                        } else {                            // both points
                            pr t = mul2s(wx[p][0], w[p]);
#pragma unroll
                            for (int a = 1; a < 4; ++a) t = fma2s(wx[p][a], w[p + a], t);
                            sb[p] = r == 1 ? mul2(WY[p][0], t) : fma2(WY[p][r - 1], t, sb[p]);
                        }
                    }
                }
#pragma unroll
                for (int p = 0; p < V; ++p) sb[p] = fma2(WE[p], pk(e0[p], e4[p]), sb[p]);
#pragma unroll
                for (int p = 0; p < V; ++p) {
                    const pr wzc = lagrange_one(c, tz[p], hz[p]);
                    sc[p] = c == 0 ? mul2(wzc, sb[p]) : fma2(wzc, sb[p], sc[p]);
                }
            }
#if STB200_TRI2_RELDEP
            release(g + o, bits32(plo(sc[0])) ^ bits32(phi(sc[0])) ^ bits32(plo(sc[V - 1])) ^ bits32(phi(sc[V - 1])));
#else
            // fenced release (pipe.cuh): the data-dependent form waited for the
            // last FMA chain of the plane and cost 3% (160 vs 165 Gpt/s SHUFFLE)
            mbar_release_fenced(&empty[(g + o) % NS]);
#endif
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float ov[V];
#pragma unroll
                for (int p = 0; p < V; ++p) ov[p] = h ? phi(sc[p]) : plo(sc[p]);
                float* op = optr + (h ? args.nx : 0);
                if (vec[h]) stg_vec(op, ov);
#pragma unroll
                for (int p = 0; p < V; ++p)
                    if (el[h][p]) op[p] = ov[p];
            }
            optr += plane;
        }
        release(g + nseg, 0u);
        release(g + nseg + 1, 0u);
        release(g + nseg + 2, 0u);
        g += nseg + 3;
    }
}

}  // namespace stb200
