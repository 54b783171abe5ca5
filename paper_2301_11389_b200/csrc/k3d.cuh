// k3d.cuh — 3-D register-cache stencil kernels for sm_100a (star-shaped
// stencils: laplacian3d7 / jacobi3d7, wave13pt, gradient, divergence).
//
// Shuffles apply to the leading (x = thread) dimension only (PAPER.md:505-507
// "We do not consider adjacent threads in non-leading dimensions"); the slow
// axes are staged by the Tensor Memory Accelerator:
//
//  * S1 map: a CTA works on columns of the grid: an x-tile of 32*V elements
//    (one 16-byte vector per lane) by kWarps3D*RY rows (RY consecutive rows
//    per consumer warp), marching along z.  Grid = at most one CTA per SM (a
//    persistent wave) with an equal number of (z part, column) items per CTA,
//    walked in lockstep chunk by chunk (LockIter) so neighbouring tiles
//    stream the same planes at the same time and share halo lines via L2; a
//    chunk boundary restarts the pipeline (2R planes).
//  * S2 plane load: a producer warp issues one TMA tensor copy
//    (cp.async.bulk.tensor.3d, SASS UTMALDG) per staged array per z-plane: the
//    box is the tile's 512-byte rows plus one 32-byte sector each side (for
//    arrays with x taps) and R halo rows in y (for arrays with y taps);
//    out-of-bounds parts are zero-filled by TMA and only ever feed masked
//    (non-interior) outputs.  NS stages in a ring, full/empty mbarriers.
//  * S3 x-neighbour taps (centre row of the plane): SHUFFLE = shfl.sync.up/down
//    by one lane; PLAIN = the neighbour lanes' elements read from the staged
//    box (LDS).
//  * S4 corner cases: lanes 0 / 31 read the R elements beyond the warp tile
//    from the staged sectors (the fallback load); tiles past
//    the grid edge are zero-filled by TMA, stores masked per element in edge
//    tiles only.
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

constexpr int kWarps3D = 15;      // consumer warps per CTA (+1 producer = 16 warps, one CTA per SM)

// S7 store paths: STG.128 from the lanes, or per-warp bulk copies of
// staged rows (cp.async.bulk).  (A third one, one TMA tensor store per
// output per CTA tile plane behind a named barrier, measured 2x slower on
// gradient; TMA tensor stores also fault on negative box coordinates, so
// the lower boundary ring has to be inside the box: DESIGN.md §5.2.)
enum StorePath { ST_STG = 0, ST_BULK = 1 };

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
    static constexpr int STORE = ST_STG;            // S7 store path (measured)
    static constexpr bool STREAM_ST = true;       // st.global.cs interior stores (measured +2-4%)
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
    static constexpr int STORE = ST_BULK;           // S7 store path (measured)
    static constexpr bool STREAM_ST = false;       // st.global.cs interior stores (measured +2-4%)
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
    static constexpr int STORE = ST_STG;            // S7 store path (measured)
    static constexpr bool STREAM_ST = false;       // st.global.cs interior stores (measured +2-4%)
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
    static constexpr int STORE = ST_STG;            // S7 store path (measured)
    static constexpr bool STREAM_ST = false;       // st.global.cs interior stores (measured +2-4%)
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

// deepest plane ring (stages) a kind may use, shared memory permitting
#ifndef STB200_NSMAX
#define STB200_NSMAX 8
#endif
#ifndef STB200_SMEM_KB
#define STB200_SMEM_KB 200
#endif

// ----------------------------------------------------------- smem layout
// CTA tile: TX = 32*V columns by TY = kWarps3D*RY = 30 rows; each consumer
// warp owns RY = 2 consecutive rows (its z queues fit the register budget of
// 16 warps per SM, 128 registers each).  The y halo is 2R/(30+2R) of the
// staged rows.
template <class Op, typename T>
struct Layout3 {
    static constexpr int V = vlen<T>(), R = Op::R, TX = 32 * V;
    static constexpr int RY = 2;
    static constexpr int TY = kWarps3D * RY;
    // x-halo boxes carry one 32-byte sector of the neighbour tiles on each
    // side (PADX elements): the warp-edge lanes' fallback reads come from
    // there.  (A 16-byte pad under L2 promotion, or a scalar global load, is
    // served as a whole 128-byte line: 50% extra traffic for 512-byte rows.)
    static constexpr int PADX = 32 / (int)sizeof(T);
    __host__ __device__ static constexpr int padx(int a) { return box_xh(Op::box(a)) ? PADX : 0; }
    __host__ __device__ static constexpr int bx(int a) { return TX + 2 * padx(a); }
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
    // output staging for the bulk (TMA) stores: one TX-wide row per
    // (warp, row, output), after the ring
    static constexpr int OUT_ROW = TX * (int)sizeof(T);
    static constexpr int out_bytes() {
        return Op::STORE == ST_BULK ? kWarps3D * RY * Op::NOUT * OUT_ROW : 0;
    }
    // stages: as many as fit in ~200 KB with the staging (one CTA per SM), at least 2R+2
    static constexpr int NS_FIT = (STB200_SMEM_KB * 1024 - out_bytes()) / stage_bytes();
    static constexpr int NS = NS_FIT > STB200_NSMAX ? STB200_NSMAX : (NS_FIT < 2 * R + 2 ? 2 * R + 2 : NS_FIT);
    static constexpr size_t out_off() { return (size_t)NS * stage_bytes(); }
    static constexpr size_t smem_bytes() {
        return out_off() + out_bytes() + 2 * NS * sizeof(uint64_t);
    }
    static_assert(smem_bytes() <= 232448, "k3d shared memory over the 227 KB per-CTA limit");
};
constexpr int k3d_threads() { return (kWarps3D + 1) * 32; }

// Work order ("lockstep round robin"): a work item is (z part, column);
// items are numbered with the column fastest and CTA c owns items c, c+G,
// c+2G, ... (m of them).  Every CTA walks its items chunk by chunk (zc planes
// of each item per round), so at any time CTA c and CTA c+1 (x-neighbour
// tiles) and CTA c+ntx (y-neighbour) stream the same z planes: the halo rows
// and edge sectors they share are fetched from DRAM once and hit L2 for the
// other.  Items per CTA are equal (the grid is sized to make them so), so
// the CTAs stay in step without any grid-wide synchronisation.
struct LockIter {
    int64_t ncols;
    int nzo, zsplit, zc, m, nchunks, chunk = 0, j = -1;
    unsigned cta, G;
    __device__ LockIter(int64_t ncols_, int nzo_, int zsplit_, int zc_, int m_, unsigned cta_, unsigned G_)
        : ncols(ncols_), nzo(nzo_), zsplit(zsplit_), zc(zc_), m(m_), cta(cta_), G(G_) {
        const int max_len = (nzo + zsplit - 1) / zsplit;
        nchunks = (max_len + zc - 1) / zc;
    }
    // next piece: column col, output planes [zo, zo + nseg) (relative to z_lo)
    __device__ __forceinline__ bool next(int64_t& col, int& zo, int& nseg) {
        for (;;) {
            if (++j == m) { j = 0; ++chunk; }
            if (chunk >= nchunks) return false;
            const int64_t item = (int64_t)cta + (int64_t)j * G;
            if (item >= ncols * zsplit) continue;
            const int zpart = (int)(item / ncols);
            col = item - (int64_t)zpart * ncols;
            const int zb = (int)((int64_t)nzo * zpart / zsplit);
            const int ze = (int)((int64_t)nzo * (zpart + 1) / zsplit);
            zo = zb + chunk * zc;
            if (zo >= ze) continue;
            nseg = ze - zo < zc ? ze - zo : zc;
            return true;
        }
    }
};

template <class Op, typename T>
struct K3Args {
    const T* in[Op::NA];   // for the warp-edge fallback loads (x halo of the tile)
    T* out[Op::NOUT];
    int64_t nx, ny;
    int z_lo, nzo;         // output planes [z_lo, z_lo + nzo)
    int ntx, nty;          // tile counts
    int zsplit, zc, m;     // LockIter: z parts per column, chunk planes, items per CTA
    PeerOut<T> peer;       // fused halo stores of out[0] (P2P multi-GPU), off when null
    int dbg;               // experiment switches (0 in production)
    int store;             // S7 path used (StorePath; the kind's compiled path or ST_STG)
};

// Experiment switches (build.build_experiment): 1 = interior-warp rows take
// a uniform STG.128-only branch (measured slower: DESIGN.md §5.2).
#ifndef STB200_XIN
#define STB200_XIN 0
#endif
// 1 = SHUFFLE edge fallback as two predicated loads (the first form)
#ifndef STB200_FB_PRED
#define STB200_FB_PRED 0
#endif
// 1 = interior stores with st.global.cs (evict-first)
#ifndef STB200_STCS
#define STB200_STCS 0
#endif

// ------------------------------------------------------------------ kernel
template <class Op, typename T, int VARIANT, bool FUSED = false>
__global__ void __launch_bounds__(k3d_threads(), 1)
k3d(const __grid_constant__ TmapPack<Op::NA> tm, const __grid_constant__ K3Args<Op, T> args,
    const Coeffs<T, Op::NC> c) {
    using L = Layout3<Op, T>;
    constexpr int R = Op::R, NA = Op::NA, V = L::V, TX = L::TX, TY = L::TY;
    constexpr int RY = L::RY, NS = L::NS, NQ = 2 * R + 1;
    constexpr bool BULK = Op::STORE == ST_BULK && !FUSED;   // bulk-store path compiled in (S7)

    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::out_off() + L::out_bytes());
    uint64_t* empty = full + NS;
    const int warp = threadIdx.x >> 5, lane = lane_id();

    const int64_t ncols = (int64_t)args.ntx * args.nty;
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
            uint32_t g = 0;                                // arrivals so far (all pieces)
            LockIter it(ncols, args.nzo, args.zsplit, args.zc, args.m, blockIdx.x, gridDim.x);
            int64_t col;
            int zo, nseg;
            while (it.next(col, zo, nseg)) {
                const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
                const int z_first = args.z_lo + zo - R;
                for (int t = 0; t < nseg + 2 * R; ++t, ++g) {
                    const uint32_t s = g % NS;
                    if (g >= NS) mbar_wait_backoff<512>(&empty[s], (g / NS - 1) & 1u);
                    mbar_arrive_expect_tx(&full[s], L::tx_bytes());
                    unsigned char* st = smem + (size_t)s * L::stage_bytes();
#pragma unroll
                    for (int a = 0; a < NA; ++a)
                        tma_load_3d(st + L::box_off(a), &tm.m[a],
                                    tx * TX - L::padx(a),
                                    ty * TY - (box_yh(Op::box(a)) ? R : 0), z_first + t, &full[s]);
                }
            }
        }
        return;
    }

    // ---- consumer warps: RY rows each
    Coeffs<T, Op::NC> cr;
#pragma unroll
    for (int t = 0; t < Op::NC; ++t) cr.c[t] = c.c[t];
    const bool lane0 = lane == 0, lane31 = lane == 31;
    T q[RY][NQ][V];                                        // z queue per row
    T* out_stage = reinterpret_cast<T*>(smem + L::out_off()) + (size_t)warp * RY * Op::NOUT * TX;
    uint32_t g = 0;
    const int64_t plane = args.nx * args.ny;

    LockIter it(ncols, args.nzo, args.zsplit, args.zc, args.m, blockIdx.x, gridDim.x);
    int64_t col;
    int zo, nseg;
    while (it.next(col, zo, nseg)) {
        const int tx = (int)(col % args.ntx), ty = (int)(col / args.ntx);
        const int64_t xl = (int64_t)tx * TX + lane * V;
        const int64_t y0 = (int64_t)ty * TY + warp * RY;  // first row of this warp
        const bool own = xl < args.nx;
        const bool x_vec = own && xl >= R && xl + V <= args.nx - R;
        bool x_el[V];
#pragma unroll
        for (int p = 0; p < V; ++p) x_el[p] = !x_vec && own && xl + p >= R && xl + p < args.nx - R;
        // warp-uniform: every lane holds a whole interior vector (all but the
        // grid-edge tiles); their rows take the STG.128-only store path
        const bool xin = __all_sync(FULL, x_vec);
        bool rows_ok[RY];                                  // output row inside the grid interior
#pragma unroll
        for (int r = 0; r < RY; ++r) rows_ok[r] = y0 + r >= R && y0 + r < args.ny - R;
        int64_t obase = ((int64_t)(args.z_lo + zo) * args.ny + y0) * args.nx + xl;
        // 16-byte aligned interior span [xa, xb) of the tile's rows (bulk stores)
        const int64_t x0 = (int64_t)tx * TX;
        const int64_t xa = ((x0 > R ? x0 : R) + V - 1) / V * V;
        const int64_t xb = ((x0 + TX < args.nx - R ? x0 + TX : args.nx - R)) / V * V;
        int64_t zcur = args.z_lo + zo;                     // output plane of the next emit
        const int np = nseg + 2 * R;

        // element offset of (row warp*RY + r + dy, lane vector + e) in array a's box
        auto off = [&](int a, int r, int dy, int e) {
            return (warp * RY + r + dy + (box_yh(Op::box(a)) ? R : 0)) * L::bx(a) + L::padx(a) + lane * V + e;
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
        // arrival: wait for the plane, push each row's queue-array centre
        // returns a run-time zero computed from the loaded centres: a release
        // right after the arrival waits for those loads (pipe.cuh mbar_release)
        const uint32_t rt_zero = (uint32_t)((uint64_t)args.nx >> 48);
        auto arrive_plane = [&](uint32_t gg, int slot, int zplane) -> uint32_t {
            (void)zplane;
            mbar_wait(&full[gg % NS], (gg / NS) & 1u);
            const T* b = stage_ptr(gg, Op::QA);
            uint32_t dep = 0;
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                ld_vec(b + off(Op::QA, r, 0, 0), q[r][slot]);
                dep ^= bits32(q[r][slot][0]);
            }
            return dep & rt_zero;
        };
        auto release = [&](uint32_t gg, uint32_t dep) { mbar_release(&empty[gg % NS], dep); };

        // in-plane taps of plane gg + compute + store the RY output rows
        auto emit = [&](uint32_t gg, int u) {
#pragma unroll
            for (int r = 0; r < RY; ++r) {
                Ctx3<T, NA, V, R> x{{}, {}, {}, q[r], u};
#pragma unroll
                for (int a = 0; a < NA; ++a) {
                    const T* b = stage_ptr(gg, a);
                    if (box_xh(Op::box(a))) {
                        T v[V];
                        ld_vec(b + off(a, r, 0, 0), v);
#pragma unroll
                        for (int k = 0; k < V; ++k) x.xw[a][R + k] = v[k];
                        if constexpr (VARIANT == 0) {
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][k] = shfl_up(v[V - R + k], 1);
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][R + V + k] = shfl_down(v[k], 1);
                            // warp edge (%out_of_range): the
                            // fallback read of the staged neighbour sector, one
                            // load whose address is lane 0's (x0-R..x0-1) or the
                            // others' (x0+TX..x0+TX+R-1: lane 31's), then selects
#if STB200_FB_PRED
                            lds_pred<T, R>(lane0, b + off(a, r, 0, -R), &x.xw[a][0]);
                            lds_pred<T, R>(lane31, b + off(a, r, 0, V), &x.xw[a][R + V]);
#else
                            T e[R];
                            {
                                const T* pe = b + (warp * RY + r + (box_yh(Op::box(a)) ? R : 0)) * L::bx(a) +
                                              L::padx(a) + (lane0 ? -R : TX);
                                if constexpr (R == 2 && sizeof(T) == 4) {
                                    const float2 t2 = *reinterpret_cast<const float2*>(pe);
                                    e[0] = t2.x; e[1] = t2.y;
                                } else {
#pragma unroll
                                    for (int k = 0; k < R; ++k) e[k] = pe[k];
                                }
                            }
#pragma unroll
                            for (int k = 0; k < R; ++k) {
                                x.xw[a][k] = lane0 ? e[k] : x.xw[a][k];
                                x.xw[a][R + V + k] = lane31 ? e[k] : x.xw[a][R + V + k];
                            }
#endif
                        } else {                          // PLAIN: neighbours' elements from smem
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][k] = b[off(a, r, 0, k - R)];
#pragma unroll
                            for (int k = 0; k < R; ++k) x.xw[a][R + V + k] = b[off(a, r, 0, V + k)];
                        }
                    }
                    if (box_yh(Op::box(a))) {
#pragma unroll
                        for (int d = 1; d <= R; ++d) {
                            ld_vec(b + off(a, r, -d, 0), x.yv[a][R - d]);
                            ld_vec(b + off(a, r, d, 0), x.yv[a][R + d - 1]);
                        }
                    }
                    if (Op::box(a) == BOX_C) ld_vec(b + off(a, r, 0, 0), x.cv[a]);
                }
                T o[Op::NOUT][V];
#pragma unroll
                for (int p = 0; p < V; ++p) {
                    T res[Op::NOUT];
                    Op::point(x, p, cr, res);
#pragma unroll
                    for (int k = 0; k < Op::NOUT; ++k) o[k][p] = res[k];
                }
                const bool row_ok = rows_ok[r];
                auto store = [&](T* op, const T* ov) {
                    if (STB200_XIN && xin && row_ok) {      // uniform branch: interior warp row
                        stg_vec(op, ov);
                    } else {
                        if (row_ok && x_vec) {
                            if (STB200_STCS || Op::STREAM_ST) stcs_vec(op, ov);
                            else stg_vec(op, ov);
                        }
#pragma unroll
                        for (int p = 0; p < V; ++p)
                            if (row_ok && x_el[p]) op[p] = ov[p];
                    }
                };
                // S7 store.  Whole interior vectors go to the warp's staging row
                // and leave as one bulk copy per row (below); lanes with a
                // partial vector (grid edge) store their interior elements.
                if (BULK && args.store == ST_BULK) {
                    if (r == 0) bulk_wait_read(lane0);           // staging rows free again
#pragma unroll
                    for (int k = 0; k < Op::NOUT; ++k) {
                        if (x_vec) st_vec_s(out_stage + (r * Op::NOUT + k) * TX + lane * V, o[k]);
#pragma unroll
                        for (int p = 0; p < V; ++p)
                            if (row_ok && x_el[p]) args.out[k][obase + r * args.nx + p] = o[k][p];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < Op::NOUT; ++k) store(args.out[k] + obase + r * args.nx, o[k]);
                }
                if constexpr (FUSED) {                     // halo planes straight to the peers
                    if (args.peer.lo && zcur < args.peer.lo_end)
                        store(args.peer.lo + obase + r * args.nx + args.peer.d_lo, o[0]);
                    if (args.peer.hi && zcur >= args.peer.hi_begin)
                        store(args.peer.hi + obase + r * args.nx + args.peer.d_hi, o[0]);
                }
            }
            // one bulk copy (cp.async.bulk, the TMA engine) per interior row
            // segment and output: the stores leave the LSU queue
            if (BULK && args.store == ST_BULK) {
                fence_proxy_async_smem();
                __syncwarp();
            }
            if (BULK && args.store == ST_BULK && lane0 && xb > xa) {
#pragma unroll
                for (int r = 0; r < RY; ++r) {
                    if (y0 + r < R || y0 + r >= args.ny - R) continue;
#pragma unroll
                    for (int k = 0; k < Op::NOUT; ++k)
                        bulk_s2g(args.out[k] + (obase - lane * V) + r * args.nx + (xa - x0),
                                 out_stage + (r * Op::NOUT + k) * TX + (xa - x0), (uint32_t)((xb - xa) * sizeof(T)));
                }
                bulk_commit();
            }
            release(gg, 0u);                               // after the stores that used every tap
            obase += plane;
            ++zcur;
        };

        // prologue: planes t = 0 .. 2R-1.  Planes t < R and t >= nseg + R
        // feed only the z queue; planes [R, nseg + R) are released by the
        // output that reads them in-plane.
#pragma unroll
        for (int t = 0; t < 2 * R; ++t) {
            const uint32_t dep = arrive_plane(g + t, t, args.z_lo + zo - R + t);
            if (t < R || t >= nseg + R) release(g + t, dep);
        }
        // main: arrival t = 2R + i, output i (in-plane plane t - R)
        int i = 0;
        for (; i + NQ <= nseg; i += NQ) {
#pragma unroll
            for (int u = 0; u < NQ; ++u) {
                const uint32_t ga = g + 2 * R + i + u;
                const uint32_t dep = arrive_plane(ga, (2 * R + u) % NQ, args.z_lo + zo + R + i + u);
                if (i + u + 2 * R >= np - R) release(ga, dep);  // last R planes: centre only
                emit(ga - R, u);
            }
        }
#pragma unroll
        for (int u = 0; u < NQ - 1; ++u) {
            if (i + u < nseg) {
                const uint32_t ga = g + 2 * R + i + u;
                const uint32_t dep = arrive_plane(ga, (2 * R + u) % NQ, args.z_lo + zo + R + i + u);
                if (i + u + 2 * R >= np - R) release(ga, dep);
                emit(ga - R, u);
            }
        }
        g += np;
    }
    if (BULK) bulk_wait_all(lane0);
}

}  // namespace stb200
