// k3d.cuh — 3-D register-cache stencil kernels for sm_100a (star-shaped
// stencils: laplacian3d7 / jacobi3d7, wave13pt, gradient, divergence).
//
// Shuffles apply to the leading (x = thread) dimension only (PAPER.md:505-507
// "We do not consider adjacent threads in non-leading dimensions"); the slow
// axes are staged by the Tensor Memory Accelerator:
//
//  * S1 map: a CTA owns a column of the grid: an x-tile of 32*V elements (one
//    16-byte vector per lane) by kWarps3D rows (one consumer warp per row),
//    and marches along z.  The (column, z) work space is linearised and cut
//    into one equal contiguous share per CTA (one wave, grid = resident CTAs
//    = a multiple of the SM count), so every CTA streams the same number of
//    planes; a share that crosses a column restarts the pipeline there.
//  * S2 plane load: a producer warp issues one TMA tensor copy
//    (cp.async.bulk.tensor.3d, SASS UTMALDG) per staged array per z-plane: the
//    box covers the tile plus a 16-byte x pad and R halo rows in y as the
//    array needs; out-of-bounds parts are zero-filled by TMA and only ever
//    feed masked (non-interior) outputs.  NS stages in a ring, full/empty
//    mbarriers per stage.
//  * S3 x-neighbour taps (centre row of the plane): SHUFFLE = shfl.sync.up/down
//    by one lane + the warp-edge fallback read from the staged box; PLAIN =
//    read from the staged box (LDS).
//  * S4 corner cases: warp-edge lanes as above; tiles past the grid edge are
//    zero-filled by TMA, stores masked per element in edge tiles only.
//  * S5 slow-axis taps: y taps are LDS.128 of the neighbour rows of the same
//    staged plane; z taps come from a per-lane register queue of the 2R+1
//    most recent planes' centre vectors (rotated by unrolling).
//  * S6 arithmetic: Op::point, identical code for both variants.
//  * S7 store: STG.128 of interior points.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "pipe.cuh"

namespace stb200 {

constexpr int kWarps3D = 8;       // consumer warps = rows of the CTA tile (Ty)

// Staged-box shapes: which halos an array's stencil needs.
enum BoxKind { BOX_XY = 0, BOX_X = 1, BOX_Y = 2, BOX_C = 3 };
__host__ __device__ constexpr bool box_xh(int b) { return b == BOX_XY || b == BOX_X; }
__host__ __device__ constexpr bool box_yh(int b) { return b == BOX_XY || b == BOX_Y; }

template <int NA>
struct TmapPack { CUtensorMap m[NA]; };

// Per-output register context handed to Op::point.
//   X(a, p, dx): array a, centre row, element p of the lane's vector, x offset dx
//   Y(a, p, dy): array a, row y+dy (dy != 0), same column
//   C(a, p):     array a at the output point (centre-only arrays)
//   Z(p, dz):    queue array at plane z+dz (dz in [-R, R])
template <typename T, int NA, int V, int R>
struct Ctx3 {
    static constexpr int NQ = 2 * R + 1;
    T xw[NA][V + 2 * R];
    T yv[NA][2 * R][V];
    T cv[NA][V];
    const T (&q)[NQ][V];
    int u;                              // unroll phase: queue slot of plane z is (u + R) % NQ
    __device__ __forceinline__ T X(int a, int p, int dx) const { return xw[a][p + R + dx]; }
    __device__ __forceinline__ T Y(int a, int p, int dy) const {
        return yv[a][dy < 0 ? R + dy : R + dy - 1][p];
    }
    __device__ __forceinline__ T C(int a, int p) const { return cv[a][p]; }
    __device__ __forceinline__ T Z(int p, int dz) const { return q[(u + R + dz) % NQ][p]; }
};

// ---------------------------------------------------------------- stencils
// Each Op: radius R, arrays NA with box kinds, queue array QA (centres feed
// the z queue), outputs NOUT, coefficients NC, point formula in the oracle's
// term order (oracle/oracle.c), evaluated in T with FMA.

// laplacian3d7 / jacobi3d7: a*C + b*(x+1 + x-1 + y+1 + y-1 + z+1 + z-1)
template <typename T> struct OpLap7 {
    static constexpr int R = 1, NA = 1, QA = 0, NOUT = 1, NC = 2;
    __host__ __device__ static constexpr int box(int) { return BOX_XY; }
    template <class Cx>
    __device__ __forceinline__ static void point(const Cx& x, int p, const Coeffs<T, NC>& c, T* o) {
        T s = x.X(0, p, 1) + x.X(0, p, -1);
        s = s + x.Y(0, p, 1);
        s = s + x.Y(0, p, -1);
        s = s + x.Z(p, 1);
        s = s + x.Z(p, -1);
        o[0] = fma(c.c[1], s, c.c[0] * x.X(0, p, 0));
    }
};

// wave13pt: m0*cur + m1*(6 at distance 1) + m2*(6 at distance 2) - prev
template <typename T> struct OpWave13 {
    static constexpr int R = 2, NA = 2, QA = 1, NOUT = 1, NC = 3;
    __host__ __device__ static constexpr int box(int a) { return a == 0 ? BOX_C : BOX_XY; }  // prev, cur
    template <class Cx>
    __device__ __forceinline__ static void point(const Cx& x, int p, const Coeffs<T, NC>& c, T* o) {
        T s1 = x.X(1, p, 1) + x.X(1, p, -1);
        s1 = s1 + x.Y(1, p, 1);
        s1 = s1 + x.Y(1, p, -1);
        s1 = s1 + x.Z(p, 1);
        s1 = s1 + x.Z(p, -1);
        T s2 = x.X(1, p, 2) + x.X(1, p, -2);
        s2 = s2 + x.Y(1, p, 2);
        s2 = s2 + x.Y(1, p, -2);
        s2 = s2 + x.Z(p, 2);
        s2 = s2 + x.Z(p, -2);
        T r = fma(c.c[1], s1, c.c[0] * x.X(1, p, 0));
        r = fma(c.c[2], s2, r);
        o[0] = r - x.C(0, p);
    }
};

// gradient: (ax*(x+1 - x-1), ay*(y+1 - y-1), az*(z+1 - z-1))
template <typename T> struct OpGradient {
    static constexpr int R = 1, NA = 1, QA = 0, NOUT = 3, NC = 3;
    __host__ __device__ static constexpr int box(int) { return BOX_XY; }
    template <class Cx>
    __device__ __forceinline__ static void point(const Cx& x, int p, const Coeffs<T, NC>& c, T* o) {
        o[0] = c.c[0] * (x.X(0, p, 1) - x.X(0, p, -1));
        o[1] = c.c[1] * (x.Y(0, p, 1) - x.Y(0, p, -1));
        o[2] = c.c[2] * (x.Z(p, 1) - x.Z(p, -1));
    }
};

// divergence: ax*(u[x+1]-u[x-1]) + ay*(v[y+1]-v[y-1]) + az*(w[z+1]-w[z-1])
template <typename T> struct OpDivergence {
    static constexpr int R = 1, NA = 3, QA = 2, NOUT = 1, NC = 3;
    __host__ __device__ static constexpr int box(int a) {  // u, v, w
        return a == 0 ? BOX_X : a == 1 ? BOX_Y : BOX_C;
    }
    template <class Cx>
    __device__ __forceinline__ static void point(const Cx& x, int p, const Coeffs<T, NC>& c, T* o) {
        T r = c.c[0] * (x.X(0, p, 1) - x.X(0, p, -1));
        r = fma(c.c[1], x.Y(1, p, 1) - x.Y(1, p, -1), r);
        o[0] = fma(c.c[2], x.Z(p, 1) - x.Z(p, -1), r);
    }
};

// ----------------------------------------------------------- smem layout
template <class Op, typename T>
struct Layout3 {
    static constexpr int V = vlen<T>(), R = Op::R, PAD = vlen<T>(), TX = 32 * V, TY = kWarps3D;
    __host__ __device__ static constexpr int bx(int a) { return TX + (box_xh(Op::box(a)) ? 2 * PAD : 0); }
    __host__ __device__ static constexpr int by(int a) { return TY + (box_yh(Op::box(a)) ? 2 * R : 0); }
    __host__ __device__ static constexpr int box_bytes(int a) { return bx(a) * by(a) * (int)sizeof(T); }
    __host__ __device__ static constexpr int box_stride(int a) { return (box_bytes(a) + 127) / 128 * 128; }
    __host__ __device__ static constexpr int box_off(int a) {
        return a == 0 ? 0 : box_off(a - 1) + box_stride(a - 1);
    }
    __host__ __device__ static constexpr int stage_bytes() { return box_off(Op::NA); }
    __host__ __device__ static constexpr int tx_bytes() {
        int s = 0;
        for (int a = 0; a < Op::NA; ++a) s += box_bytes(a);
        return s;
    }
    static constexpr int NS = R == 1 ? 4 : 6;              // pipeline stages
    static constexpr size_t smem_bytes() { return (size_t)NS * stage_bytes() + 2 * NS * sizeof(uint64_t); }
};
constexpr int k3d_threads() { return (kWarps3D + 1) * 32; }

template <class Op, typename T>
struct K3Args {
    T* out[Op::NOUT];
    int64_t nx, ny;
    int z_lo, nzo;         // output planes [z_lo, z_lo + nzo)
    int ntx, nty;          // tile counts
    int64_t work;          // ntx * nty * nzo
};

// ------------------------------------------------------------------ kernel
template <class Op, typename T, int VARIANT>
__global__ void __launch_bounds__(k3d_threads())
k3d(const __grid_constant__ TmapPack<Op::NA> tm, const __grid_constant__ K3Args<Op, T> args,
    const Coeffs<T, Op::NC> c) {
    using L = Layout3<Op, T>;
    constexpr int R = Op::R, NA = Op::NA, V = L::V, PAD = L::PAD, TX = L::TX, NS = L::NS;
    constexpr int NQ = 2 * R + 1;

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * L::stage_bytes());
    uint64_t* empty = full + NS;
    const int warp = threadIdx.x >> 5, lane = lane_id();

    // this CTA's share of the linearised (column, z) work
    const int64_t G = gridDim.x;
    const int64_t w_begin = args.work * (int64_t)blockIdx.x / G;
    const int64_t w_end = args.work * ((int64_t)blockIdx.x + 1) / G;
    if (w_begin >= w_end) return;                          // CTA-uniform

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps3D * 32);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kWarps3D) {                                // ---- producer warp
        if (lane == 0) {
            for (int a = 0; a < NA; ++a) prefetch_tmap(&tm.m[a]);
            uint32_t g = 0;                                // arrivals so far (all segments)
            for (int64_t w = w_begin; w < w_end;) {
                const int64_t col = w / args.nzo;
                const int zo = (int)(w - col * args.nzo);
                const int nseg = (int)(args.nzo - zo < w_end - w ? args.nzo - zo : w_end - w);
                const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
                const int z_first = args.z_lo + zo - R;
                for (int t = 0; t < nseg + 2 * R; ++t, ++g) {
                    const uint32_t s = g % NS;
                    if (g >= NS) mbar_wait(&empty[s], (g / NS - 1) & 1u);
                    mbar_arrive_expect_tx(&full[s], L::tx_bytes());
                    unsigned char* st = smem + (size_t)s * L::stage_bytes();
#pragma unroll
                    for (int a = 0; a < NA; ++a)
                        tma_load_3d(st + L::box_off(a), &tm.m[a],
                                    tx * TX - (box_xh(Op::box(a)) ? PAD : 0),
                                    ty * kWarps3D - (box_yh(Op::box(a)) ? R : 0), z_first + t,
                                    &full[s]);
                }
                w += nseg;
            }
        }
        return;
    }

    // ---- consumer warps: one row each
    Coeffs<T, Op::NC> cr;
#pragma unroll
    for (int t = 0; t < Op::NC; ++t) cr.c[t] = c.c[t];
    const bool lane0 = lane == 0, lane31 = lane == 31;
    T q[NQ][V];
    uint32_t g = 0;

    for (int64_t w = w_begin; w < w_end;) {
        const int64_t col = w / args.nzo;
        const int zo = (int)(w - col * args.nzo);
        const int nseg = (int)(args.nzo - zo < w_end - w ? args.nzo - zo : w_end - w);
        const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
        const int64_t xl = (int64_t)tx * TX + lane * V;
        const int64_t y = (int64_t)ty * kWarps3D + warp;
        const bool row_ok = y >= R && y < args.ny - R;
        const bool own = xl < args.nx;
        const bool vec_store = row_ok && own && xl >= R && xl + V <= args.nx - R;
        bool el_store[V];
#pragma unroll
        for (int p = 0; p < V; ++p)
            el_store[p] = row_ok && !vec_store && own && xl + p >= R && xl + p < args.nx - R;
        const int64_t plane = args.nx * args.ny;
        int64_t obase = ((int64_t)(args.z_lo + zo) * args.ny + y) * args.nx + xl;
        const int np = nseg + 2 * R;

        // element offset of (row warp+dy, lane vector + e) inside array a's box
        auto off = [&](int a, int dy, int e) {
            return (warp + dy + (box_yh(Op::box(a)) ? R : 0)) * L::bx(a) +
                   (box_xh(Op::box(a)) ? PAD : 0) + lane * V + e;
        };
        auto stage_ptr = [&](uint32_t gg, int a) {
            return reinterpret_cast<const T*>(smem + (size_t)(gg % NS) * L::stage_bytes() + L::box_off(a));
        };
        auto ld_vec = [&](const T* p, T* v) {
            using VT = typename VecOf<T>::type;
            const VT t = *reinterpret_cast<const VT*>(p);
            if constexpr (V == 4) { v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
            else { v[0] = t.x; v[1] = t.y; }
        };
        // arrival: wait for the plane, push the queue array's centre
        auto arrive_plane = [&](uint32_t gg, T* qslot) {
            mbar_wait(&full[gg % NS], (gg / NS) & 1u);
            ld_vec(stage_ptr(gg, Op::QA) + off(Op::QA, 0, 0), qslot);
        };
        auto release = [&](uint32_t gg) { mbar_arrive(&empty[gg % NS]); };

        // in-plane taps of plane gg + compute + store output at obase
        auto emit = [&](uint32_t gg, int u) {
            Ctx3<T, NA, V, R> x{{}, {}, {}, q, u};
#pragma unroll
            for (int a = 0; a < NA; ++a) {
                const T* b = stage_ptr(gg, a);
                {
                    if (box_xh(Op::box(a))) {
                        T v[V];
                        ld_vec(b + off(a, 0, 0), v);
#pragma unroll
                        for (int k = 0; k < V; ++k) x.xw[a][R + k] = v[k];
                        if constexpr (VARIANT == 0) {
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][k] = shfl_up(v[V - R + k], 1);
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][R + V + k] = shfl_down(v[k], 1);
                            const int e = lane0 ? -R : V;
                            T hv[R];
#pragma unroll
                            for (int k = 0; k < R; ++k) hv[k] = b[off(a, 0, e + k)];
#pragma unroll
                            for (int k = 0; k < R; ++k) {
                                x.xw[a][k] = lane0 ? hv[k] : x.xw[a][k];
                                x.xw[a][R + V + k] = lane31 ? hv[k] : x.xw[a][R + V + k];
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][k] = b[off(a, 0, k - R)];
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][R + V + k] = b[off(a, 0, V + k)];
                        }
                    }
                    if (box_yh(Op::box(a))) {
#pragma unroll
                        for (int d = 1; d <= R; ++d) {
                            ld_vec(b + off(a, -d, 0), x.yv[a][R - d]);
                            ld_vec(b + off(a, d, 0), x.yv[a][R + d - 1]);
                        }
                    }
                    if (Op::box(a) == BOX_C) ld_vec(b + off(a, 0, 0), x.cv[a]);
                }
            }
            T o[Op::NOUT][V];
#pragma unroll
            for (int p = 0; p < V; ++p) {
                T r[Op::NOUT];
                Op::point(x, p, cr, r);
#pragma unroll
                for (int k = 0; k < Op::NOUT; ++k) o[k][p] = r[k];
            }
            release(gg);
#pragma unroll
            for (int k = 0; k < Op::NOUT; ++k) {
                T* op = args.out[k] + obase;
                if (vec_store) stg_vec(op, o[k]);
#pragma unroll
                for (int p = 0; p < V; ++p)
                    if (el_store[p]) op[p] = o[k][p];
            }
            obase += plane;
        };

        // prologue: planes t = 0 .. 2R-1.  Planes t < R and t >= nseg + R
        // feed only the z queue; planes [R, nseg + R) are released by the
        // output that reads them in-plane.
#pragma unroll
        for (int t = 0; t < 2 * R; ++t) {
            arrive_plane(g + t, q[t]);
            if (t < R || t >= nseg + R) release(g + t);
        }
        // main: arrival t = 2R + i, output i (in-plane plane t - R)
        int i = 0;
        for (; i + NQ <= nseg; i += NQ) {
#pragma unroll
            for (int u = 0; u < NQ; ++u) {
                const uint32_t ga = g + 2 * R + i + u;
                arrive_plane(ga, q[(2 * R + u) % NQ]);
                if (i + u + 2 * R >= np - R) release(ga);  // last R planes: centre only
                emit(ga - R, u);
            }
        }
#pragma unroll
        for (int u = 0; u < NQ - 1; ++u) {
            if (i + u < nseg) {
                const uint32_t ga = g + 2 * R + i + u;
                arrive_plane(ga, q[(2 * R + u) % NQ]);
                if (i + u + 2 * R >= np - R) release(ga);
                emit(ga - R, u);
            }
        }
        g += np;
        w += nseg;
    }
}

}  // namespace stb200
