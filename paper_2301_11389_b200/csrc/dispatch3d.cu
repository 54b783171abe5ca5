// dispatch3d.cu — host launchers of the 3-D kernels (k3d.cuh): TMA tensor
// maps (cuTensorMapEncodeTiled through the runtime's driver entry point, no
// libcuda link), one-wave grid sizing, variant selection.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "k3d.cuh"
#include "ktricubic.cuh"
#include "ktricubic2.cuh"
#include "kpaper3d.cuh"
#include "kgrad.cuh"
#include "klap2.cuh"

namespace stb200 {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D tensor map over a dense (nz, ny, nx) array, box (bx, by, 1), zero OOB fill.
static cudaError_t make_tmap(CUtensorMap* m, const void* base, int dtype, const int64_t* ld, int bx, int by) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const size_t es = dtype == ST_F64 ? 8 : 4;
    cuuint64_t gdim[3] = {(cuuint64_t)ld[0], (cuuint64_t)ld[1], (cuuint64_t)ld[2]};
    cuuint64_t gstride[2] = {(cuuint64_t)ld[0] * es, (cuuint64_t)(ld[0] * ld[1]) * es};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, dtype == ST_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int sm_count_of(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return 148;
    if (!cached[device]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        cached[device] = n > 0 ? n : 148;
    }
    return cached[device];
}

template <class Op, typename T, int VAR, bool FUSED = false>
static cudaError_t launch_k3d(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                              int64_t z_lo, int64_t z_hi) {
    using L = Layout3<Op, T>;
    if (!FUSED && (h->peer_lo || h->peer_hi)) return launch_k3d<Op, T, VAR, true>(h, in, out, s, z_lo, z_hi);
    auto kern = k3d<Op, T, VAR, FUSED>;
    constexpr size_t smem = L::smem_bytes();
    const int blocks_per_sm = kernel_setup((const void*)kern, h->device, smem, k3d_threads());
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = Op::R; z_hi = ld[2] - Op::R; }
    if (z_hi <= z_lo) return cudaSuccess;
    TmapPack<Op::NA> tm;
    for (int a = 0; a < Op::NA; ++a) {
        cudaError_t e = make_tmap(&tm.m[a], in[a], h->dtype, ld, L::bx(a), L::by(a));
        if (e != cudaSuccess) return e;
    }
    K3Args<Op, T> args;
    for (int a = 0; a < Op::NA; ++a) args.in[a] = (const T*)in[a];
    for (int k = 0; k < Op::NOUT; ++k) args.out[k] = (T*)out[k];
    args.nx = ld[0];
    args.ny = ld[1];
    args.z_lo = (int)z_lo;
    args.nzo = (int)(z_hi - z_lo);
    args.ntx = (int)((ld[0] + L::TX - 1) / L::TX);
    args.nty = (int)((ld[1] + L::TY - 1) / L::TY);
    // lockstep round robin (k3d.cuh LockIter): split z only when there are
    // fewer columns than SMs; equal items per CTA; chunks of zc planes
    const int64_t ncols = (int64_t)args.ntx * args.nty;
    const int64_t slots = (int64_t)blocks_per_sm * sm_count_of(h->device);
    int64_t zsplit = slots / ncols;
    if (zsplit < 1) zsplit = 1;
    if (zsplit > args.nzo) zsplit = args.nzo;
    const int64_t items = ncols * zsplit;
    const int64_t m = (items + slots - 1) / slots;
    const int64_t grid = (items + m - 1) / m;
    args.zsplit = (int)zsplit;
    args.m = (int)m;
    args.peer.lo = (T*)h->peer_lo;
    args.peer.hi = (T*)h->peer_hi;
    args.peer.lo_end = h->peer_lo_end;
    args.peer.hi_begin = h->peer_hi_begin;
    args.peer.d_lo = h->peer_d_lo;
    args.peer.d_hi = h->peer_d_hi;
    static const int dbg_zc = getenv("STB200_3D_ZC") ? atoi(getenv("STB200_3D_ZC")) : 0;
    // chunk depth (measured): the single-array radius-1 kinds
    // run 13-17% faster with 6-plane chunks (tighter lockstep) despite the
    // 2 restart planes per chunk; the others prefer long chunks
    // (single-array radius-1 kinds: 6-plane chunks for fp32, 4 for fp64 —
    // laplacian fp64 512^3 339 -> 377 Gpt/s, jacobi3d fp32 prefers 6)
    args.zc = dbg_zc > 0 ? dbg_zc : (Op::R == 1 && Op::NA == 1 && Op::NOUT == 1) ? (sizeof(T) == 8 ? 4 : 6) : 64;
    static const int dbg = getenv("STB200_DBG") ? atoi(getenv("STB200_DBG")) : 0;
    args.dbg = dbg;
    // S7 store path (k3d.cuh): the kind's measured choice;
    // STB200_STG=1 forces plain STG stores (A/B experiments)
    static const int stg_env = getenv("STB200_STG") ? atoi(getenv("STB200_STG")) : 0;
    args.store = stg_env ? ST_STG : Op::STORE;
    Coeffs<T, Op::NC> c{};
    for (int t = 0; t < Op::NC; ++t) c.c[t] = (T)h->coeffs[t];
    kern<<<(unsigned)grid, k3d_threads(), smem, s>>>(tm, args, c);
    return cudaGetLastError();
}

template <template <typename> class OpT, typename T>
static cudaError_t launch3_var(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                               int64_t a, int64_t b) {
    if (h->variant == ST_PLAIN) return launch_k3d<OpT<T>, T, 1>(h, in, out, s, a, b);
    return launch_k3d<OpT<T>, T, 0>(h, in, out, s, a, b);
}

cudaError_t launch_tricubic(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                            int64_t z_lo, int64_t z_hi);

// gradient (kgrad.cuh): grid (x tiles, row groups of kGradWarps, z chunks of
// zc planes).  The fused peer-store path stays on k3d (it carries PeerOut).
template <typename T, int VAR>
static cudaError_t launch_kgrad(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                                int64_t z_lo, int64_t z_hi) {
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = 1; z_hi = ld[2] - 1; }
    if (z_hi <= z_lo || ld[1] < 3 || ld[0] < 3) return cudaSuccess;
    constexpr int TX = 32 * VecOf<T>::V;
    GradArgs<T> a{};
    a.u = (const T*)in[0];
    for (int k = 0; k < 3; ++k) a.out[k] = (T*)out[k];
    a.nx = ld[0];
    a.ny = ld[1];
    a.z_lo = (int)z_lo;
    a.nzo = (int)(z_hi - z_lo);
    static const int zc_env = getenv("STB200_GRAD_ZC") ? atoi(getenv("STB200_GRAD_ZC")) : 0;
    a.zc = zc_env > 0 ? zc_env : 8;   // measured: 32 -> 8 planes 311 -> 325 Gpt/s
    for (int k = 0; k < 3; ++k) a.c[k] = (T)h->coeffs[k];
    const int64_t nzc = (a.nzo + a.zc - 1) / a.zc;
    const int64_t nyb = (ld[1] - 2 + kGradWarps - 1) / kGradWarps;
    if (nyb > 65535 || nzc > 65535) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)((ld[0] + TX - 1) / TX), (unsigned)nyb, (unsigned)nzc);
    kgrad<T, VAR><<<grid, kGradWarps * 32, 0, s>>>(a);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_gradient(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                                   int64_t a, int64_t b) {
    static const int old = getenv("STB200_GRAD_K3D") ? atoi(getenv("STB200_GRAD_K3D")) : 0;
    if (old || h->peer_lo || h->peer_hi) return launch3_var<OpGradient, T>(h, in, out, s, a, b);
    if (h->variant == ST_PLAIN) return launch_kgrad<T, 1>(h, in, out, s, a, b);
    return launch_kgrad<T, 0>(h, in, out, s, a, b);
}

// The paper-literal family for the 3-D kinds (kpaper3d.cuh): one output per
// thread, 512 threads per block along x, one block per (x block, row, plane).
template <int KIND, int PV>
static cudaError_t launch_kpaper3d(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                                   int64_t z_lo, int64_t z_hi) {
    const int64_t* ld = h->ldims;
    const int lo = h->k->lo, hi = h->k->hi;
    if (z_lo < 0) { z_lo = lo; z_hi = ld[2] - hi; }
    if (z_hi <= z_lo) return cudaSuccess;
    const int64_t rows = ld[1] - lo - hi;
    if (rows > 65535 || z_hi - z_lo > 65535) return cudaErrorInvalidConfiguration;
    P3Args a{};
    for (int t = 0; t < h->k->n_in; ++t) a.in[t] = (const uint32_t*)in[t];
    for (int t = 0; t < h->k->n_out; ++t) a.out[t] = (float*)out[t];
    a.nx = ld[0];
    a.ny = ld[1];
    a.z_lo = (int)z_lo;
    a.lo = lo;
    a.hi = hi;
    for (int t = 0; t < 3 && t < h->k->ncoeffs; ++t) a.c[t] = (float)h->coeffs[t];
    const dim3 grid((unsigned)((ld[0] - lo - hi + kPaperThreads - 1) / kPaperThreads), (unsigned)rows,
                    (unsigned)(z_hi - z_lo));
    kpaper3d<KIND, PV><<<grid, kPaperThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int KIND>
static cudaError_t paper3_var(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                              int64_t a, int64_t b) {
    switch (h->variant) {
    case ST_PAPER_ORIGINAL: return launch_kpaper3d<KIND, PV_ORIGINAL>(h, in, out, s, a, b);
    case ST_PAPER_PTXASW: return launch_kpaper3d<KIND, PV_PTXASW>(h, in, out, s, a, b);
    case ST_PAPER_NOLOAD: return launch_kpaper3d<KIND, PV_NOLOAD>(h, in, out, s, a, b);
    case ST_PAPER_NOCORNER: return launch_kpaper3d<KIND, PV_NOCORNER>(h, in, out, s, a, b);
    default: return launch_kpaper3d<KIND, PV_UNIFORM>(h, in, out, s, a, b);
    }
}

// lapgsrb (klap2.cuh): one-wave persistent grid, LockIter work order as k3d
template <typename T, int VAR>
static cudaError_t launch_lap2(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                               int64_t z_lo, int64_t z_hi) {
    using L = LapLayout<T>;
    auto kern = klapgsrb2<T, VAR>;
    const int bps = kernel_setup((const void*)kern, h->device, L::SMEM, klap2_threads());
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = 1; z_hi = ld[2] - 1; }
    if (z_hi <= z_lo) return cudaSuccess;
    TmapPack<1> tm;
    Lap2Args<T> args{};
    args.out = (T*)out[0];
    args.nx = ld[0];
    args.ny = ld[1];
    args.nz = ld[2];
    args.z_lo = (int)z_lo;
    args.nzo = (int)(z_hi - z_lo);
    args.ntx = (int)((ld[0] + L::TX - 1) / L::TX);
    const int64_t slots = (int64_t)bps * sm_count_of(h->device);
    // tile height: the even ty <= TY that maximises (useful rows of the
    // tiles) x (staged rows that are outputs, ty / (ty + 4)) x (busy SMs of
    // the one-wave grid); e.g. 1024 rows x 4 x-tiles -> ty = 28: 37 x 4 =
    // 148 columns on 148 SMs instead of 35 x 4 = 140 at ty = 30
    static const int ty_env = getenv("STB200_LAP_TY") ? atoi(getenv("STB200_LAP_TY")) : 0;
    double best = -1.0;
    int64_t best_zsplit = 1, best_m = 1;
    for (int ty = L::TY; ty >= 8; ty -= 2) {
        if (ty_env > 0 && ty != ty_env) continue;
        const int64_t nty = (ld[1] + ty - 1) / ty;
        const int64_t ncols = (int64_t)args.ntx * nty;
        int64_t zsplit = slots / ncols;
        if (zsplit < 1) zsplit = 1;
        if (zsplit > args.nzo) zsplit = args.nzo;
        const int64_t items = ncols * zsplit;
        const int64_t m = (items + slots - 1) / slots;
        const double rows_eff = (double)(ld[1] - 2) / (double)(nty * ty);
        const double stage_eff = (double)ty / (ty + 4);
        const double util = (double)items / (double)(m * slots);
        const double score = rows_eff * stage_eff * util;
        if (score > best + 1e-9) {
            best = score;
            args.ty = ty;
            args.nty = (int)nty;
            best_zsplit = zsplit;
            best_m = m;
        }
    }
    if (best < 0) return cudaErrorInvalidValue;
    const int64_t items = (int64_t)args.ntx * args.nty * best_zsplit;
    const int64_t grid = (items + best_m - 1) / best_m;
    args.zsplit = (int)best_zsplit;
    args.m = (int)best_m;
    static const int zc_env = getenv("STB200_LAP_ZC") ? atoi(getenv("STB200_LAP_ZC")) : 0;
    args.zc = zc_env > 0 ? zc_env : 64;
    args.w = (T)h->coeffs[0];
    cudaError_t e = make_tmap(&tm.m[0], in[0], h->dtype, ld, L::BX, args.ty + 4);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, klap2_threads(), L::SMEM, s>>>(tm, args);
    return cudaGetLastError();
}

cudaError_t dispatch_f3(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s, int64_t a,
                        int64_t b);

cudaError_t dispatch_3d(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                        int64_t a, int64_t b) {
    const bool f64 = h->dtype == ST_F64;
    if (h->variant >= ST_PAPER_ORIGINAL) {                 // validated fp32 in set_variant
        switch (h->k->kind) {
        case ST_LAPLACIAN3D7:
        case ST_JACOBI3D7: return paper3_var<1>(h, in, out, s, a, b);
        case ST_WAVE13PT: return paper3_var<2>(h, in, out, s, a, b);
        case ST_DIVERGENCE: return paper3_var<3>(h, in, out, s, a, b);
        case ST_GRADIENT: return paper3_var<4>(h, in, out, s, a, b);
        case ST_TRICUBIC: return paper3_var<5>(h, in, out, s, a, b);
        default: return cudaErrorInvalidValue;
        }
    }
    switch (h->k->kind) {
    case ST_LAPLACIAN3D7:
    case ST_JACOBI3D7:
        return f64 ? launch3_var<OpLap7, double>(h, in, out, s, a, b)
                   : launch3_var<OpLap7, float>(h, in, out, s, a, b);
    case ST_WAVE13PT:
        return f64 ? launch3_var<OpWave13, double>(h, in, out, s, a, b)
                   : launch3_var<OpWave13, float>(h, in, out, s, a, b);
    case ST_GRADIENT:
        return f64 ? launch_gradient<double>(h, in, out, s, a, b)
                   : launch_gradient<float>(h, in, out, s, a, b);
    case ST_DIVERGENCE:
        return f64 ? launch3_var<OpDivergence, double>(h, in, out, s, a, b)
                   : launch3_var<OpDivergence, float>(h, in, out, s, a, b);
    case ST_TRICUBIC:
    case ST_TRICUBIC2:       // the same function up to rounding order (DESIGN.md §3 R19)
        return launch_tricubic(h, in, out, s, a, b);
    case ST_LAPGSRB: {
        // klapgsrb2 (klap2.cuh, default); STB200_LAP1=1 selects the first
        // z-marching kernel klapgsrb (kf3.cuh) for A/B experiments
        static const int old1 = getenv("STB200_LAP1") ? atoi(getenv("STB200_LAP1")) : 0;
        if (old1) return dispatch_f3(h, in, out, s, a, b);
        if (f64) return h->variant == ST_PLAIN ? launch_lap2<double, 1>(h, in, out, s, a, b)
                                               : launch_lap2<double, 0>(h, in, out, s, a, b);
        return h->variant == ST_PLAIN ? launch_lap2<float, 1>(h, in, out, s, a, b)
                                      : launch_lap2<float, 0>(h, in, out, s, a, b);
    }
    case ST_UXX1: return dispatch_f3(h, in, out, s, a, b);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace stb200

namespace stb200 {

template <typename T, int VAR>
static cudaError_t launch_tri(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                              int64_t z_lo, int64_t z_hi) {
    using L = TriLayout<T>;
    auto kern = ktricubic<T, VAR>;
    kernel_setup((const void*)kern, h->device, L::SMEM, (kTriWarps + 1) * 32);
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = 1; z_hi = ld[2] - 2; }
    if (z_hi <= z_lo) return cudaSuccess;
    TmapPack<1> tm;
    cudaError_t e = make_tmap(&tm.m[0], in[0], h->dtype, ld, L::FBX, L::FBY);
    if (e != cudaSuccess) return e;
    TriArgs<T> args;
    args.X = (const T*)in[1];
    args.Y = (const T*)in[2];
    args.Z = (const T*)in[3];
    args.out = (T*)out[0];
    args.nx = ld[0];
    args.ny = ld[1];
    args.z_lo = (int)z_lo;
    args.nzo = (int)(z_hi - z_lo);
    args.ntx = (int)((ld[0] + L::TX - 1) / L::TX);
    args.nty = (int)((ld[1] + L::TY - 1) / L::TY);
    const int64_t ncols = (int64_t)args.ntx * args.nty;
    const int64_t slots = sm_count_of(h->device);
    int64_t zsplit = slots / ncols;
    if (zsplit < 1) zsplit = 1;
    if (zsplit > args.nzo) zsplit = args.nzo;
    const int64_t items = ncols * zsplit;
    const int64_t m = (items + slots - 1) / slots;
    const int64_t grid = (items + m - 1) / m;
    args.zsplit = (int)zsplit;
    args.m = (int)m;
    args.zc = 64;
    kern<<<(unsigned)grid, (kTriWarps + 1) * 32, L::SMEM, s>>>(tm, args);
    return cudaGetLastError();
}

// fp32: two output rows per warp, flattened equal ranges (ktricubic2.cuh)
template <int VAR>
static cudaError_t launch_tri2(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                               int64_t z_lo, int64_t z_hi) {
    using L = Tri2Layout;
    auto kern = ktricubic2<VAR>;
    kernel_setup((const void*)kern, h->device, L::SMEM, (kTri2Warps + 1) * 32);
    const int64_t* ld = h->ldims;
    if (z_lo < 0) { z_lo = 1; z_hi = ld[2] - 2; }
    if (z_hi <= z_lo) return cudaSuccess;
    TmapPack<4> tm;
    cudaError_t e = make_tmap(&tm.m[0], in[0], h->dtype, ld, L::FBX, L::FBY);
    for (int a = 1; a < 4 && e == cudaSuccess; ++a) e = make_tmap(&tm.m[a], in[a], h->dtype, ld, L::TX, L::TY);
    if (e != cudaSuccess) return e;
    TriArgs<float> args{};
    args.X = (const float*)in[1];
    args.Y = (const float*)in[2];
    args.Z = (const float*)in[3];
    args.out = (float*)out[0];
    args.nx = ld[0];
    args.ny = ld[1];
    args.z_lo = (int)z_lo;
    args.nzo = (int)(z_hi - z_lo);
    args.ntx = (int)((ld[0] + L::TX - 1) / L::TX);
    args.nty = (int)((ld[1] + L::TY - 1) / L::TY);
    const int64_t items = (int64_t)args.ntx * args.nty * args.nzo;
    int64_t grid = sm_count_of(h->device);
    if (grid > items) grid = items;
    kern<<<(unsigned)grid, (kTri2Warps + 1) * 32, L::SMEM, s>>>(tm, args);
    return cudaGetLastError();
}

cudaError_t launch_tricubic(const stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                            int64_t a, int64_t b) {
    // fp32: ktricubic2 (default); STB200_TRI1=1 selects the one-row
    // ktricubic (A/B experiments)
    static const int old1 = getenv("STB200_TRI1") ? atoi(getenv("STB200_TRI1")) : 0;
    if (h->dtype == ST_F32 && !old1)
        return h->variant == ST_PLAIN ? launch_tri2<1>(h, in, out, s, a, b) : launch_tri2<0>(h, in, out, s, a, b);
    if (h->dtype == ST_F64)
        return h->variant == ST_PLAIN ? launch_tri<double, 1>(h, in, out, s, a, b)
                                      : launch_tri<double, 0>(h, in, out, s, a, b);
    return h->variant == ST_PLAIN ? launch_tri<float, 1>(h, in, out, s, a, b)
                                  : launch_tri<float, 0>(h, in, out, s, a, b);
}

}  // namespace stb200
