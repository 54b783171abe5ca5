// dispatch2d.cu — host launchers of the 2-D kernels (k2d.cuh).
#include <cstdlib>

#include "internal.h"
#include "k2d.cuh"
#include "kpaper.cuh"
#include "ktb2d.cuh"
#include "ktb2r.cuh"
#include "k2d2.cuh"
#include "klife.cuh"

namespace stb200 {

// coefficient t of Op: the factored gaussblur weights for the separable op
template <class Op>
static double op_coeff(const stencil_s* h, int t) {
    return IsSep<Op>::value ? h->gsep_c[t] : h->coeffs[t];
}

static int sm_count(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return 148;
    if (!cached[device]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        cached[device] = n > 0 ? n : 148;
    }
    return cached[device];
}

// Strip height: short strips of kStripH output rows, many waves of CTAs.
// Measured on B200: with blocks dispatched in blockIdx
// order, the rows being streamed at any moment form one contiguous band of
// the grid (good DRAM row locality, and the 2R rows two neighbouring strips
// share are read once, from L2, by the second); one wave of tall strips
// scatters the accesses over ~40 bands and ran 13-30% slower.
// FUSED: the P2P instantiation with the peer halo stores (a separate kernel,
// so the plain path carries none of its registers or branches).
template <class Op, typename T, int VAR, bool FUSED = false>
static cudaError_t launch_k2d(const stencil_s* h, const void* in, void* out, cudaStream_t s,
                              int64_t y_lo, int64_t y_hi) {
    constexpr int R = Op::R;
    constexpr int V = vlen<T>();
    constexpr int kStripH = 24;
    if (!FUSED && (h->peer_lo || h->peer_hi)) return launch_k2d<Op, T, VAR, true>(h, in, out, s, y_lo, y_hi);
    auto kern = k2d<Op, T, VAR, FUSED>;
    constexpr size_t smem = k2d_smem_bytes<T>();
    kernel_setup((const void*)kern, h->device, smem, k2d_threads());
    const int64_t nx = h->ldims[0], ny = h->ldims[1];
    if (y_lo < 0) { y_lo = R; y_hi = ny - R; }
    if (y_hi <= y_lo) return cudaSuccess;
    const int64_t ntiles = (nx + 32 * V - 1) / (32 * V);
    const int64_t gx = (ntiles + kWarps2D - 1) / kWarps2D;
    const int64_t rows = y_hi - y_lo;
    static const int dbg_h = getenv("STB200_2D_H") ? atoi(getenv("STB200_2D_H")) : 0;
    // small grids: shorter strips so that at least ~2 CTAs per SM exist
    int64_t H = (rows * gx + 2 * sm_count(h->device) - 1) / (2 * sm_count(h->device));
    H = H < 4 ? 4 : H > kStripH ? kStripH : H;
    if (dbg_h > 0) H = dbg_h;
    const int64_t nstrips = (rows + H - 1) / H;
    if (nstrips > 65535) return cudaErrorInvalidConfiguration;
    Coeffs<T, Op::NC> c{};
    for (int t = 0; t < Op::NC; ++t) c.c[t] = (T)op_coeff<Op>(h, t);
    PeerOut<T> peer;
    peer.lo = (T*)h->peer_lo;
    peer.hi = (T*)h->peer_hi;
    peer.lo_end = h->peer_lo_end;
    peer.hi_begin = h->peer_hi_begin;
    peer.d_lo = h->peer_d_lo;
    peer.d_hi = h->peer_d_hi;
    kern<<<dim3((unsigned)gx, (unsigned)nstrips), k2d_threads(), smem, s>>>(
        (const T*)in, (T*)out, nx, (int)y_lo, (int)y_hi, (int)H, c, peer);
    return cudaGetLastError();
}

template <template <typename> class OpT, typename T>
static cudaError_t launch_var(const stencil_s* h, const void* in, void* out, cudaStream_t s,
                              int64_t a, int64_t b) {
    if (h->variant == ST_PLAIN) return launch_k2d<OpT<T>, T, VAR_PLAIN>(h, in, out, s, a, b);
    return launch_k2d<OpT<T>, T, VAR_SHUFFLE>(h, in, out, s, a, b);
}

// The paper-literal family (kpaper.cuh): one output per thread, 512 threads
// per block along x, one block row per output row.
template <typename T, int KIND, int PV>
static cudaError_t launch_kpaper(const stencil_s* h, const void* in, void* out, cudaStream_t s,
                                 int64_t y_lo, int64_t y_hi) {
    constexpr int R = PaperOp<T, KIND>::R;
    const int64_t nx = h->ldims[0], ny = h->ldims[1];
    if (y_lo < 0) { y_lo = R; y_hi = ny - R; }
    if (y_hi <= y_lo) return cudaSuccess;
    if (y_hi - y_lo > 65535) return cudaErrorInvalidConfiguration;
    Coeffs<T, PaperOp<T, KIND>::NC> c{};
    for (int t = 0; t < PaperOp<T, KIND>::NC; ++t) c.c[t] = (T)h->coeffs[t];
    const dim3 grid((unsigned)((nx - 2 * R + kPaperThreads - 1) / kPaperThreads), (unsigned)(y_hi - y_lo));
    kpaper<T, KIND, PV><<<grid, kPaperThreads, 0, s>>>((const T*)in, (T*)out, nx, (int)y_lo, c);
    return cudaGetLastError();
}

template <typename T, int KIND>
static cudaError_t paper_var(const stencil_s* h, const void* in, void* out, cudaStream_t s, int64_t a,
                             int64_t b) {
    switch (h->variant) {
    case ST_PAPER_ORIGINAL: return launch_kpaper<T, KIND, PV_ORIGINAL>(h, in, out, s, a, b);
    case ST_PAPER_PTXASW: return launch_kpaper<T, KIND, PV_PTXASW>(h, in, out, s, a, b);
    case ST_PAPER_NOLOAD: return launch_kpaper<T, KIND, PV_NOLOAD>(h, in, out, s, a, b);
    case ST_PAPER_NOCORNER: return launch_kpaper<T, KIND, PV_NOCORNER>(h, in, out, s, a, b);
    default: return launch_kpaper<T, KIND, PV_UNIFORM>(h, in, out, s, a, b);
    }
}

cudaError_t dispatch_f3(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s, int64_t a,
                        int64_t b);

cudaError_t dispatch_2d(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                        int64_t a, int64_t b) {
    const bool f64 = h->dtype == ST_F64;
    if (h->variant >= ST_PAPER_ORIGINAL) {                 // validated f32/i32 in set_variant
        switch (h->k->kind) {
        case ST_JACOBI2D5: return paper_var<float, 1>(h, in[0], out[0], s, a, b);
        case ST_JACOBI2D9: return paper_var<float, 2>(h, in[0], out[0], s, a, b);
        case ST_GAUSSBLUR5X5: return paper_var<float, 3>(h, in[0], out[0], s, a, b);
        case ST_GAMEOFLIFE: return paper_var<int, 4>(h, in[0], out[0], s, a, b);
        default: return cudaErrorInvalidValue;
        }
    }
    switch (h->k->kind) {
    case ST_JACOBI2D5:
        return f64 ? launch_var<OpJacobi2D5, double>(h, in[0], out[0], s, a, b)
                   : launch_var<OpJacobi2D5, float>(h, in[0], out[0], s, a, b);
    case ST_JACOBI2D9:
        return f64 ? launch_var<OpJacobi2D9, double>(h, in[0], out[0], s, a, b)
                   : launch_var<OpJacobi2D9, float>(h, in[0], out[0], s, a, b);
    case ST_GAUSSBLUR5X5:
        if (h->gsep)
            return f64 ? launch_var<OpGauss5Sep, double>(h, in[0], out[0], s, a, b)
                       : launch_var<OpGauss5Sep, float>(h, in[0], out[0], s, a, b);
        return f64 ? launch_var<OpGauss5, double>(h, in[0], out[0], s, a, b)
                   : launch_var<OpGauss5, float>(h, in[0], out[0], s, a, b);
    case ST_GAMEOFLIFE:
        if (h->variant == ST_PLAIN) return launch_k2d<OpLife, int, VAR_PLAIN>(h, in[0], out[0], s, a, b);
        return launch_k2d<OpLife, int, VAR_SHUFFLE>(h, in[0], out[0], s, a, b);
    case ST_WHISPERING: return dispatch_f3(h, in, out, s, a, b);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace stb200

namespace stb200 {

// Temporally blocked launch: S sweeps in one kernel (ktb2d.cuh).
template <class Op, typename T>
static cudaError_t launch_tb(const stencil_s* h, const void* in, void* out, cudaStream_t s, int S) {
    constexpr int R = Op::R;
    const int64_t nx = h->ldims[0], ny = h->ldims[1];
    const int hh = S * R;
    const size_t smem = 2 * (size_t)(kTbTileX + 2 * hh) * (kTbTileY + 2 * hh) * sizeof(T);
    kernel_setup((const void*)ktb2d<Op, T>, h->device, smem, kTbThreads);
    const dim3 grid((unsigned)((nx - 2 * R + kTbTileX - 1) / kTbTileX),
                    (unsigned)((ny - 2 * R + kTbTileY - 1) / kTbTileY));
    Coeffs<T, Op::NC> c{};
    for (int t = 0; t < Op::NC; ++t) c.c[t] = (T)op_coeff<Op>(h, t);
    ktb2d<Op, T><<<grid, kTbThreads, smem, s>>>((const T*)in, (T*)out, (int)nx, (int)ny, S, c);
    return cudaGetLastError();
}

// Two sweeps per launch, streaming (k2d2.cuh): the large-grid form of
// temporal blocking.  Strips of H sweep-2 rows in blockIdx order, as k2d.
template <class Op, typename T, int VAR, int NSW>
static cudaError_t launch_k2d2(const stencil_s* h, const void* in, void* out, cudaStream_t s) {
    constexpr int R = Op::R;
    // strip height (measured): the extra input rows of a
    // strip amortise over tall strips — jacobi2d5 32768^2 fp32 1302 (24) ->
    // 1459 (128) Gpt/s, flat to 512; fp64 16384^2 best at 48-64
    constexpr int kStripH = sizeof(T) == 8 ? 64 : 128;
    auto kern = k2d2<Op, T, VAR, NSW>;
    constexpr int NW = k2d2_nw<Op, T, VAR, NSW>();
    constexpr size_t smem = k2d2_smem_bytes<T, NSW, NW, k2d2_stages<R, T>()>();
    kernel_setup((const void*)kern, h->device, smem, k2d2_threads<NW>());
    const int64_t nx = h->ldims[0], ny = h->ldims[1];
    const int64_t y_lo = R, y_hi = ny - R;
    if (y_hi <= y_lo) return cudaSuccess;
    const int64_t gx = (nx + NW * k2d2_txo<T, NSW>() - 1) / (NW * k2d2_txo<T, NSW>());
    const int64_t rows = y_hi - y_lo;
    static const int dbg_h = getenv("STB200_2D2_H") ? atoi(getenv("STB200_2D2_H")) : 0;
    int64_t H = (rows * gx + 2 * sm_count(h->device) - 1) / (2 * sm_count(h->device));
    H = H < 4 ? 4 : H > kStripH ? kStripH : H;
    if (dbg_h > 0) H = dbg_h;
    const int64_t nstrips = (rows + H - 1) / H;
    if (nstrips > 65535 || ny > INT32_MAX) return cudaErrorInvalidConfiguration;
    Coeffs<T, Op::NC> c{};
    for (int t = 0; t < Op::NC; ++t) c.c[t] = (T)op_coeff<Op>(h, t);
    kern<<<dim3((unsigned)gx, (unsigned)nstrips), k2d2_threads<NW>(), smem, s>>>(
        (const T*)in, (T*)out, nx, (int)ny, (int)y_lo, (int)y_hi, (int)H, c);
    return cudaGetLastError();
}

// All S sweeps of a small run in one launch, the field in registers (ktb2r.cuh).
template <class Op, typename T, int VAR>
static cudaError_t launch_tbr(const stencil_s* h, const void* in, void* out, cudaStream_t s, int S) {
    constexpr int R = Op::R;
    const int64_t nx = h->ldims[0], ny = h->ldims[1];
    const int hh = S * R;
    const int ow = tbr_width<T>() - 2 * hh - (kTbrV - 1), oh = kTbrWarps * kTbrRows - 2 * hh;
    auto kern = ktb2r<Op, T, VAR>;
    constexpr size_t smem = tbr_smem_bytes<T, R, VAR>();
    kernel_setup((const void*)kern, h->device, smem, kTbrWarps * 32);
    const dim3 grid((unsigned)((nx - 2 * R + ow - 1) / ow), (unsigned)((ny - 2 * R + oh - 1) / oh));
    Coeffs<T, Op::NC> c{};
    for (int t = 0; t < Op::NC; ++t) c.c[t] = (T)op_coeff<Op>(h, t);
    kern<<<grid, kTbrWarps * 32, smem, s>>>((const T*)in, (T*)out, (int)nx, (int)ny, S, c);
    return cudaGetLastError();
}

// S sweeps in one launch: the register kernel (ktb2r) when its region holds
// the S*R halo, else the shared-memory tile kernel (ktb2d).
template <class Op, typename T>
static cudaError_t launch_fused(const stencil_s* h, const void* in, void* out, cudaStream_t s, int S) {
    static const int env_old = getenv("STB200_TB_SMEM") ? atoi(getenv("STB200_TB_SMEM")) : 0;
    if (!env_old && S <= tbr_max_sweeps<T>(Op::R))
        return h->variant == ST_PLAIN ? launch_tbr<Op, T, VAR_PLAIN>(h, in, out, s, S)
                                      : launch_tbr<Op, T, VAR_SHUFFLE>(h, in, out, s, S);
    return launch_tb<Op, T>(h, in, out, s, S);
}

// gameoflife, packed four cells per register (klife.cuh); launch geometry as launch_k2d2
template <int VAR, int NSW>
static cudaError_t launch_life(const stencil_s* h, const void* in, void* out, cudaStream_t s) {
    constexpr int kStripH = 128;
    auto kern = k2dlife<VAR, NSW>;
    constexpr size_t smem = k2d2_smem_bytes<int, NSW, kWarpsLife>();
    kernel_setup((const void*)kern, h->device, smem, k2d2_threads<kWarpsLife>());
    const int64_t nx = h->ldims[0], ny = h->ldims[1];
    const int64_t y_lo = 1, y_hi = ny - 1;
    if (y_hi <= y_lo) return cudaSuccess;
    const int64_t gx = (nx + kWarpsLife * k2d2_txo<int, NSW>() - 1) / (kWarpsLife * k2d2_txo<int, NSW>());
    const int64_t rows = y_hi - y_lo;
    static const int dbg_h = getenv("STB200_2D2_H") ? atoi(getenv("STB200_2D2_H")) : 0;
    int64_t H = (rows * gx + 2 * sm_count(h->device) - 1) / (2 * sm_count(h->device));
    H = H < 4 ? 4 : H > kStripH ? kStripH : H;
    if (dbg_h > 0) H = dbg_h;
    const int64_t nstrips = (rows + H - 1) / H;
    if (nstrips > 65535 || ny > INT32_MAX) return cudaErrorInvalidConfiguration;
    kern<<<dim3((unsigned)gx, (unsigned)nstrips), k2d2_threads<kWarpsLife>(), smem, s>>>(
        (const int*)in, (int*)out, nx, (int)ny, (int)y_lo, (int)y_hi, (int)H);
    return cudaGetLastError();
}

template <class Op, typename T>
static cudaError_t pair_op(const stencil_s* h, const void* in, void* out, cudaStream_t s, int nsw) {
    // gameoflife: the packed kernel (klife.cuh); STB200_LIFE_INT=1 selects
    // the int32 k2d2 form for A/B runs
    static const int life_int = getenv("STB200_LIFE_INT") ? atoi(getenv("STB200_LIFE_INT")) : 0;
    if constexpr (std::is_same<Op, OpLife>::value) {
        if (!life_int) {
            if (h->variant == ST_PLAIN)
                return nsw == 3 ? launch_life<VAR_PLAIN, 3>(h, in, out, s) : launch_life<VAR_PLAIN, 2>(h, in, out, s);
            return nsw == 3 ? launch_life<VAR_SHUFFLE, 3>(h, in, out, s) : launch_life<VAR_SHUFFLE, 2>(h, in, out, s);
        }
    }
    if (h->variant == ST_PLAIN)
        return nsw == 3 ? launch_k2d2<Op, T, VAR_PLAIN, 3>(h, in, out, s) : launch_k2d2<Op, T, VAR_PLAIN, 2>(h, in, out, s);
    return nsw == 3 ? launch_k2d2<Op, T, VAR_SHUFFLE, 3>(h, in, out, s) : launch_k2d2<Op, T, VAR_SHUFFLE, 2>(h, in, out, s);
}

// nsw sweeps (2 or 3) in one streaming launch (k2d2.cuh)
cudaError_t dispatch_2d_pair(stencil_s* h, const void* in, void* out, cudaStream_t s, int nsw) {
    const bool f64 = h->dtype == ST_F64;
    switch (h->k->kind) {
    case ST_JACOBI2D5:
        return f64 ? pair_op<OpJacobi2D5<double>, double>(h, in, out, s, nsw)
                   : pair_op<OpJacobi2D5<float>, float>(h, in, out, s, nsw);
    case ST_JACOBI2D9:
        return f64 ? pair_op<OpJacobi2D9<double>, double>(h, in, out, s, nsw)
                   : pair_op<OpJacobi2D9<float>, float>(h, in, out, s, nsw);
    case ST_GAUSSBLUR5X5:   // two sweeps only (issue-bound already at two)
        if (h->gsep)   // separable: two or three sweeps per launch
            return f64 ? pair_op<OpGauss5Sep<double>, double>(h, in, out, s, nsw)
                       : pair_op<OpGauss5Sep<float>, float>(h, in, out, s, nsw);
        if (h->variant == ST_PLAIN)
            return f64 ? launch_k2d2<OpGauss5<double>, double, VAR_PLAIN, 2>(h, in, out, s)
                       : launch_k2d2<OpGauss5<float>, float, VAR_PLAIN, 2>(h, in, out, s);
        return f64 ? launch_k2d2<OpGauss5<double>, double, VAR_SHUFFLE, 2>(h, in, out, s)
                   : launch_k2d2<OpGauss5<float>, float, VAR_SHUFFLE, 2>(h, in, out, s);
    case ST_GAMEOFLIFE: return pair_op<OpLife, int>(h, in, out, s, nsw);
    default: return cudaErrorInvalidValue;
    }
}

// Largest fusion depth: the register kernel's (ktb2r), or the shared-memory
// tile kernel's (two planes in ~100 KB) when STB200_TB_SMEM selects it.
int fused_max_sweeps(const stencil_s* h) {
    const int R = h->k->lo;
    static const int env_old = getenv("STB200_TB_SMEM") ? atoi(getenv("STB200_TB_SMEM")) : 0;
    if (!env_old) return h->dtype == ST_F64 ? tbr_max_sweeps<double>(R) : tbr_max_sweeps<float>(R);
    const size_t es = h->dtype == ST_F64 ? 8 : 4;
    int S = 16;
    while (S > 1 && 2 * (size_t)(kTbTileX + 2 * S * R) * (kTbTileY + 2 * S * R) * es > 100 * 1024) --S;
    return S;
}

cudaError_t dispatch_2d_fused(stencil_s* h, const void* in, void* out, cudaStream_t s, int S) {
    const bool f64 = h->dtype == ST_F64;
    switch (h->k->kind) {
    case ST_JACOBI2D5:
        return f64 ? launch_fused<OpJacobi2D5<double>, double>(h, in, out, s, S)
                   : launch_fused<OpJacobi2D5<float>, float>(h, in, out, s, S);
    case ST_JACOBI2D9:
        return f64 ? launch_fused<OpJacobi2D9<double>, double>(h, in, out, s, S)
                   : launch_fused<OpJacobi2D9<float>, float>(h, in, out, s, S);
    case ST_GAUSSBLUR5X5:
        if (h->gsep)
            return f64 ? launch_fused<OpGauss5Sep<double>, double>(h, in, out, s, S)
                       : launch_fused<OpGauss5Sep<float>, float>(h, in, out, s, S);
        return f64 ? launch_fused<OpGauss5<double>, double>(h, in, out, s, S)
                   : launch_fused<OpGauss5<float>, float>(h, in, out, s, S);
    case ST_GAMEOFLIFE: return launch_fused<OpLife, int>(h, in, out, s, S);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace stb200
