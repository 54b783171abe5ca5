// ktb2r.cuh — register-resident temporal blocking for small 2-D grids
// (BASELINE configs[0], jacobi 512^2 x 10): all S
// sweeps of a run in ONE launch, the field held in registers between sweeps.
//
// A 512^2 fp32 grid is 1 MiB: a sweep is ~0.1 us of work spread over the GPU
// and a run of 10 sweeps is bound by launch latency and by how fast each SM
// gets through its sweeps.  Here a CTA owns a region of 32*V columns (V
// elements per lane, one 8- or 16-byte vector) by NW*RB rows (RB
// consecutive rows per warp), loads it once, applies S sweeps in registers
// and stores its output tile — the region minus a halo of h = S*R cells on
// every side, which the neighbouring CTAs recompute (the invalid margin
// grows by R per sweep, so after S sweeps it is exactly the halo).
//
// Per sweep a cell needs its R neighbours:
//   x  SHUFFLE: shfl.up / shfl.down of the neighbour lane's edge elements
//      (a lane at the region edge reads garbage that only
//      feeds the invalid margin: no corner case);
//      PLAIN: the warp's rows go through shared memory and the R neighbour
//      elements are loaded (LDS) by every lane;
//   y  the rows above / below the warp's RB rows are the neighbour warps'
//      edge rows, exchanged through shared memory with one __syncthreads per
//      sweep (double-buffered slots).
// Cells on the global boundary ring (and outside the grid) are held: the
// Dirichlet rule of stencil_run.  Every updated cell goes through Op::point
// of k2d.cuh on the same operands, so the result is bit-identical to S
// single sweeps.  Edge tiles also store the ring cells next to them (as
// ktb2d): a fused run needs no separate ring copy.
#pragma once
#include "common.cuh"
#include "k2d.cuh"

namespace stb200 {

#ifndef STB200_TBR_NW
#define STB200_TBR_NW 16          // warps per CTA
#endif
#ifndef STB200_TBR_RB
#define STB200_TBR_RB 4           // rows per warp
#endif
#ifndef STB200_TBR_V
#define STB200_TBR_V 2            // elements per lane: region = 32*V columns
#endif
constexpr int kTbrWarps = STB200_TBR_NW, kTbrRows = STB200_TBR_RB, kTbrV = STB200_TBR_V;

// Regions of 64 x 64 cells (V = 2, 16 warps x 4 rows): 144 CTAs for a 512^2
// grid at S = 10 (one per SM), against 95 of 128 x 48 with V = 4 (measured:
// DESIGN.md §5.4).
template <typename T>
__host__ __device__ constexpr int tbr_width() { return 32 * kTbrV; }

// Largest S the region supports for radius R: the output tile keeps >= 16
// columns and >= 8 rows.
template <typename T>
__host__ __device__ constexpr int tbr_max_sweeps(int R) {
    const int sx = (tbr_width<T>() - 16 - (kTbrV - 1)) / (2 * R);
    const int sy = (kTbrWarps * kTbrRows - 8) / (2 * R);
    return sx < sy ? sx : sy;
}

// V-element vectors (V = 1, 2, 4; 4, 8 or 16 bytes) in global and shared memory
template <typename T, int V> struct VecN;
template <typename T> struct VecN<T, 1> { using type = T; };
template <> struct VecN<float, 2> { using type = float2; };
template <> struct VecN<int, 2> { using type = int2; };
template <> struct VecN<double, 2> { using type = double2; };
template <> struct VecN<float, 4> { using type = float4; };
template <> struct VecN<int, 4> { using type = int4; };
template <int V, typename T>
__device__ __forceinline__ void vld(T* v, const T* p) {
    const typename VecN<T, V>::type t = *reinterpret_cast<const typename VecN<T, V>::type*>(p);
    const T* q = reinterpret_cast<const T*>(&t);
#pragma unroll
    for (int e = 0; e < V; ++e) v[e] = q[e];
}
template <int V, typename T>
__device__ __forceinline__ void vldg(T* v, const T* p) {
    const typename VecN<T, V>::type t = __ldg(reinterpret_cast<const typename VecN<T, V>::type*>(p));
    const T* q = reinterpret_cast<const T*>(&t);
#pragma unroll
    for (int e = 0; e < V; ++e) v[e] = q[e];
}
template <int V, typename T>
__device__ __forceinline__ void vst(T* p, const T* v) {
    typename VecN<T, V>::type t;
    T* q = reinterpret_cast<T*>(&t);
#pragma unroll
    for (int e = 0; e < V; ++e) q[e] = v[e];
    *reinterpret_cast<typename VecN<T, V>::type*>(p) = t;
}

// Window over the register rows of one warp: rows -R .. RB-1+R (neighbour
// warps' rows at the ends), elements -R .. V-1+R of this lane's columns.
template <typename T, int V, int R>
struct RegWin {
    const T (&rows)[kTbrRows + 2 * R][V + 2 * R];
    int r;                                  // output row (0 .. RB-1)
    __device__ __forceinline__ T operator()(int dj, int e) const { return rows[r + R + dj][e]; }
};

// Dynamic shared memory: per warp R top and R bottom rows, two parities
// (edge), and for PLAIN the warp's own RB rows (stage); every row padded by
// 4 elements on each side so that the lanes at the region edge read pad.
template <typename T> __host__ __device__ constexpr int tbr_pitch() { return tbr_width<T>() + 8; }
template <typename T, int R, int VAR>
__host__ __device__ constexpr size_t tbr_smem_bytes() {
    return (size_t)(2 * kTbrWarps * 2 * R + (VAR == VAR_PLAIN ? kTbrWarps * kTbrRows : 0)) * tbr_pitch<T>() * sizeof(T);
}

// One sweep of a warp's RB register rows (helper of ktb2r): exchange the edge
// rows, gather the window, apply Op::point; MASK = hold the cells outside the
// grid interior (CTAs whose region touches the boundary ring).
template <class Op, typename T, int VAR, bool MASK, int V>
__device__ __forceinline__ void tbr_sweep(T (&a)[kTbrRows][V], uint32_t upd, T* mine, const T* above,
                                          const T* below, T* stage, const Coeffs<T, Op::NC>& c) {
    // mine / above / below: this warp's and the neighbour warps' 2R edge rows
    // of this sweep's parity, at this lane's columns; stage: this warp's RB
    // staged rows (PLAIN)
    constexpr int R = Op::R, RB = kTbrRows, NR = RB + 2 * R, P = tbr_pitch<T>();
    // publish the R top and R bottom rows of this warp
#pragma unroll
    for (int t = 0; t < R; ++t) {
        vst<V>(mine + t * P, a[t]);
        vst<V>(mine + (R + t) * P, a[RB - R + t]);
    }
    if (VAR == VAR_PLAIN) {
        __syncwarp();                                    // this warp's reads of its staged rows are done
#pragma unroll
        for (int r = 0; r < RB; ++r) vst<V>(stage + r * P, a[r]);
    }
    __syncthreads();
    T w[NR][V + 2 * R];
    // rows above / below: the neighbour warps' edge rows (warp 0's upper and
    // warp NW-1's lower neighbours are outside the region: margin cells)
#pragma unroll
    for (int t = 0; t < R; ++t) {
        T v[V];
        vld<V>(v, above + (R + t) * P);
#pragma unroll
        for (int e = 0; e < V; ++e) w[t][R + e] = v[e];
        vld<V>(v, below + t * P);
#pragma unroll
        for (int e = 0; e < V; ++e) w[R + RB + t][R + e] = v[e];
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int e = 0; e < V; ++e) w[R + r][R + e] = a[r][e];
    // x halos of every window row (R elements each side of the lane's vector)
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        if (VAR == VAR_SHUFFLE) {
#pragma unroll
            for (int t = 0; t < R; ++t) {
                // element -R+t of this lane is element V-R+t of the left lane;
                // element V+t is element t of the right lane (V >= R)
                w[q][t] = shfl_up(w[q][V + t], 1);
                w[q][R + V + t] = shfl_down(w[q][R + t], 1);
            }
        } else {                                        // PLAIN: loads of the staged rows
            const T* row = q < R ? above + (R + q) * P : q >= R + RB ? below + (q - R - RB) * P
                                                                      : stage + (q - R) * P;
#pragma unroll
            for (int t = 0; t < R; ++t) {
                w[q][t] = row[t - R];
                w[q][R + V + t] = row[V + t];
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const RegWin<T, V, R> win{w, r};
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const T v = Op::point(win, e, c);
            a[r][e] = (!MASK || (upd >> (r * V + e) & 1u)) ? v : a[r][e];
        }
    }
}

template <class Op, typename T, int VAR>
__global__ void __launch_bounds__(kTbrWarps * 32)
ktb2r(const T* __restrict__ in, T* __restrict__ out, int nx, int ny, int S, Coeffs<T, Op::NC> c) {
    constexpr int R = Op::R, V = kTbrV, W = 32 * V, RB = kTbrRows, NW = kTbrWarps;
    static_assert(V >= R, "the x halo comes from the neighbour lane only");
    constexpr int P = tbr_pitch<T>();
    extern __shared__ __align__(16) unsigned char smem_tbr[];
    T* const edge_base = reinterpret_cast<T*>(smem_tbr);                  // [2][NW][2R][P]
    T* const stage_base = edge_base + 2 * NW * 2 * R * P;                 // [NW][RB][P] (PLAIN)
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int h = S * R;
    // output tile [ox0, ox0 + ow) x [oy0, oy0 + oh); the region starts h cells
    // before it, rounded down to a whole vector (hence ow = W - 2h - (V-1))
    const int ow = W - 2 * h - (V - 1), oh = NW * RB - 2 * h;
    const int ox0 = R + (int)blockIdx.x * ow, oy0 = R + (int)blockIdx.y * oh;
    const int gx0 = ox0 - h >= 0 ? (ox0 - h) / V * V : -(((h - ox0) + V - 1) / V) * V;
    const int gy0 = oy0 - h;
    const int cx = gx0 + lane * V;                       // this lane's first column
    const int ry = gy0 + warp * RB;                      // this warp's first row

    // load the region (cells outside the grid: 0, never stored)
    T a[RB][V];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int gy = ry + r;
        const bool rowok = gy >= 0 && gy < ny;
        if (rowok && cx >= 0 && cx + V <= nx) {
            vldg<V>(a[r], in + (size_t)gy * nx + cx);
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e)
                a[r][e] = rowok && cx + e >= 0 && cx + e < nx ? in[(size_t)gy * nx + cx + e] : T(0);
        }
    }
    // edge-row slots of this warp and its neighbours (parity 0; parity 1 is
    // PSTRIDE further), at this lane's columns
    constexpr int PSTRIDE = NW * 2 * R * P;
    const int up = warp > 0 ? warp - 1 : 0, dn = warp < NW - 1 ? warp + 1 : NW - 1;
    T* const mine = edge_base + warp * 2 * R * P + 4 + lane * V;
    const T* const above = edge_base + up * 2 * R * P + 4 + lane * V;
    const T* const below = edge_base + dn * 2 * R * P + 4 + lane * V;
    T* const stage = stage_base + warp * RB * P + 4 + lane * V;
    // a region inside the grid interior updates every cell (no selects)
    const bool inner = gx0 >= R && gx0 + W <= nx - R && gy0 >= R && gy0 + NW * RB <= ny - R;
    if (inner) {
        int s = 0;
        for (; s + 1 < S; s += 2) {
            tbr_sweep<Op, T, VAR, false, V>(a, 0u, mine, above, below, stage, c);
            tbr_sweep<Op, T, VAR, false, V>(a, 0u, mine + PSTRIDE, above + PSTRIDE, below + PSTRIDE, stage, c);
        }
        if (s < S) tbr_sweep<Op, T, VAR, false, V>(a, 0u, mine, above, below, stage, c);
    } else {
        // cells updated by a sweep: interior of the global grid (bit r*V+e)
        uint32_t upd = 0;
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const int gx = cx + e, gy = ry + r;
                if (gx >= R && gx < nx - R && gy >= R && gy < ny - R) upd |= 1u << (r * V + e);
            }
        int s = 0;
        for (; s + 1 < S; s += 2) {
            tbr_sweep<Op, T, VAR, true, V>(a, upd, mine, above, below, stage, c);
            tbr_sweep<Op, T, VAR, true, V>(a, upd, mine + PSTRIDE, above + PSTRIDE, below + PSTRIDE, stage, c);
        }
        if (s < S) tbr_sweep<Op, T, VAR, true, V>(a, upd, mine, above, below, stage, c);
    }
    // store the output tile (and the ring cells next to an edge tile)
    const bool left = blockIdx.x == 0, right = blockIdx.x == gridDim.x - 1;
    const bool top = blockIdx.y == 0, bottom = blockIdx.y == gridDim.y - 1;
    const int tx0 = left ? 0 : ox0, tx1 = right ? nx : ox0 + ow;
    const int ty0 = top ? 0 : oy0, ty1 = bottom ? ny : oy0 + oh;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int gy = ry + r;
        if (gy < ty0 || gy >= ty1 || gy >= ny) continue;
        if (cx >= tx0 && cx + V <= tx1 && cx + V <= nx) {
            vst<V>(out + (size_t)gy * nx + cx, a[r]);
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const int gx = cx + e;
                if (gx >= tx0 && gx < tx1 && gx < nx && gx >= 0) out[(size_t)gy * nx + gx] = a[r][e];
            }
        }
    }
}

}  // namespace stb200
