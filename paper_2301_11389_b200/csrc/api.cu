// api.cu — the C ABI of include/stencil.h: validation, dispatch to the
// sm_100a kernels, Dirichlet ring copy, CUDA-graph capture of stencil_run,
// host-buffer end-to-end entry point.  Multi-GPU plumbing is in dist.cu.
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/stencil.h"
#include "internal.h"

using namespace stb200;

// ----------------------------------------------------------------- errors
static thread_local std::string g_last_error;

int stb200::set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

extern "C" const char* stencil_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* stencil_version(void) {
    return "stencil_b200 0.1 (sm_100a register-cache stencils, arxiv 2301.11389 hot path)";
}

// ------------------------------------------------------------ kind table
const KindInfo* stb200::kind_info(int kind) {
    // kind, name, ndims, n_in, n_out, lo, hi, ncoeffs, iterable(1 pingpong, 2 wave), allow_f, allow_i
    static const KindInfo table[] = {
        {ST_JACOBI2D5, "jacobi2d5", 2, 1, 1, 1, 1, 2, 1, true, false},
        {ST_JACOBI2D9, "jacobi2d9", 2, 1, 1, 1, 1, 3, 1, true, false},
        {ST_GAUSSBLUR5X5, "gaussblur5x5", 2, 1, 1, 2, 2, 25, 1, true, false},
        {ST_GAMEOFLIFE, "gameoflife", 2, 1, 1, 1, 1, 0, 1, false, true},
        {ST_LAPLACIAN3D7, "laplacian3d7", 3, 1, 1, 1, 1, 2, 1, true, false},
        {ST_JACOBI3D7, "jacobi3d7", 3, 1, 1, 1, 1, 2, 1, true, false},
        {ST_WAVE13PT, "wave13pt", 3, 2, 1, 2, 2, 3, 2, true, false},
        {ST_DIVERGENCE, "divergence", 3, 3, 1, 1, 1, 3, 0, true, false},
        {ST_GRADIENT, "gradient", 3, 1, 3, 1, 1, 3, 0, true, false},
        {ST_TRICUBIC, "tricubic", 3, 4, 1, 1, 2, 0, 0, true, false},
        {ST_TRICUBIC2, "tricubic2", 3, 4, 1, 1, 2, 0, 0, true, false},
        {ST_UXX1, "uxx1", 3, 5, 1, 2, 1, 3, 0, true, false},
        {ST_LAPGSRB, "lapgsrb", 3, 1, 1, 1, 1, 1, 1, true, false},
        {ST_WHISPERING, "whispering", 2, 8, 3, 1, 1, 0, 0, true, false},
    };
    for (const auto& k : table)
        if (k.kind == kind) return &k;
    return nullptr;
}

// Default coefficients (DESIGN.md §3 R2), written independently of oracle/.
static void default_coeffs(int kind, double* c) {
    switch (kind) {
    case ST_JACOBI2D5: c[0] = 0.0; c[1] = 0.25; break;
    case ST_JACOBI2D9: c[0] = 0.25; c[1] = 0.125; c[2] = 0.0625; break;
    case ST_GAUSSBLUR5X5: {
        const double b[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
        for (int r = 0; r < 5; ++r)
            for (int q = 0; q < 5; ++q) c[r * 5 + q] = b[r] * b[q];
        break;
    }
    case ST_LAPLACIAN3D7: c[0] = -6.0; c[1] = 1.0; break;
    case ST_JACOBI3D7: c[0] = 0.0; c[1] = 1.0 / 6.0; break;
    case ST_WAVE13PT: {
        const double lambda = 1.0 / 8.0;       // Courant number squared
        c[0] = 2.0 - 7.5 * lambda;
        c[1] = (4.0 / 3.0) * lambda;
        c[2] = -lambda / 12.0;
        break;
    }
    case ST_DIVERGENCE:
    case ST_GRADIENT: c[0] = c[1] = c[2] = 0.5; break;
    case ST_UXX1: c[0] = 0.25; c[1] = 9.0 / 8.0; c[2] = -1.0 / 24.0; break;   // dth, 4th-order stagger
    case ST_LAPGSRB: c[0] = 1.0 / 6.0; break;                                  // Gauss-Seidel weight
    default: break;
    }
}

int stb200::kernel_setup(const void* func, int device, size_t smem, int threads) {
    struct Entry { size_t smem; int bps; };
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, Entry> done;
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({func, device});
    if (it != done.end() && it->second.smem >= smem) return it->second.bps;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int bps = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, func, threads, smem) != cudaSuccess || bps < 1)
        bps = 1;
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
    done[{func, device}] = Entry{smem, bps};
    return bps;
}

static size_t dtype_size(int dt) { return dt == ST_F64 ? 8 : 4; }

// ------------------------------------------------------------- lifecycle
// gaussblur5x5: if the 25 weights are rank 1 (w[dj][di] = u[dj] * v[di]
// within 1e-12 of the largest weight, e.g. the default binomial), store
// (u, v) for the separable kernels (k2d.cuh OpGauss5Sep).  Pivot: the
// largest |w|; u = its column, v = its row / pivot.  STB200_GAUSS_FULL=1
// keeps the 25-tap form (A/B experiments).
static void gauss_factor(stencil_s* h) {
    static const int full = getenv("STB200_GAUSS_FULL") ? atoi(getenv("STB200_GAUSS_FULL")) : 0;
    const double* w = h->coeffs;
    int pr = 0, pc = 0;
    double m = 0.0;
    for (int t = 0; t < 25; ++t)
        if (fabs(w[t]) > m) { m = fabs(w[t]); pr = t / 5; pc = t % 5; }
    h->gsep = false;
    if (full || m == 0.0) return;
    double u[5], v[5];
    for (int d = 0; d < 5; ++d) {
        u[d] = w[d * 5 + pc];
        v[d] = w[pr * 5 + d] / w[pr * 5 + pc];
    }
    for (int t = 0; t < 25; ++t)
        if (fabs(u[t / 5] * v[t % 5] - w[t]) > 1e-12 * m) return;
    for (int d = 0; d < 5; ++d) {
        h->gsep_c[d] = u[d];
        h->gsep_c[5 + d] = v[d];
    }
    h->gsep = true;
}

extern "C" int stencil_create(stencil_t* out, int kind, int ndims, const int64_t* dims,
                              int dtype, const double* coeffs, int ncoeffs) {
    if (!out || !dims) return set_error(ST_EARG, "null argument");
    *out = nullptr;
    const KindInfo* k = kind_info(kind);
    if (!k) return set_error(ST_EARG, "unknown kind %d", kind);
    if (dtype != ST_F32 && dtype != ST_F64 && dtype != ST_I32)
        return set_error(ST_EARG, "unknown dtype %d", dtype);
    if ((dtype == ST_I32 && !k->allow_i) || (dtype != ST_I32 && !k->allow_f))
        return set_error(ST_EUNSUPPORTED, "dtype %d not supported for %s", dtype, k->name);
    if (ndims != k->ndims) return set_error(ST_EARG, "%s needs ndims=%d", k->name, k->ndims);
    for (int d = 0; d < ndims; ++d)
        if (dims[d] < k->lo + k->hi + 1)
            return set_error(ST_EARG, "axis %d extent %lld < lo+hi+1", d, (long long)dims[d]);
    if (ncoeffs != 0 && ncoeffs != k->ncoeffs)
        return set_error(ST_EARG, "%s takes %d coefficients, got %d", k->name, k->ncoeffs, ncoeffs);
    if (ncoeffs && !coeffs) return set_error(ST_EARG, "null coeffs");
    if ((dims[0] * (int64_t)dtype_size(dtype)) % 16 != 0)
        return set_error(ST_EALIGN, "nx*sizeof(T) = %lld is not a multiple of 16 bytes",
                         (long long)(dims[0] * (int64_t)dtype_size(dtype)));
    if (dims[0] > (int64_t)1 << 30 || dims[1] > (int64_t)1 << 30 ||
        (ndims == 3 && dims[2] > (int64_t)1 << 30))
        return set_error(ST_EARG, "extent too large");

    stencil_s* h = new stencil_s();
    h->k = k;
    h->dtype = dtype;
    h->ndims = ndims;
    for (int d = 0; d < 3; ++d) h->dims[d] = d < ndims ? dims[d] : 1;
    for (int d = 0; d < 3; ++d) h->ldims[d] = h->dims[d];
    if (ncoeffs) memcpy(h->coeffs, coeffs, sizeof(double) * ncoeffs);
    else default_coeffs(kind, h->coeffs);
    h->variant = ST_SHUFFLE;
    if (kind == ST_GAUSSBLUR5X5) gauss_factor(h);
    if (cudaGetDevice(&h->device) != cudaSuccess) {
        delete h;
        return set_error(ST_ECUDA, "cudaGetDevice failed (no CUDA device?)");
    }
    *out = h;
    return ST_OK;
}

// ST_AUTO: the register-cache variant measured faster on B200 for the kind
// (profiles/r02_bench_all.txt, one session, 10 steps at the benchmark sizes,
// Gpt/s SHUFFLE vs PLAIN); a difference within 2% goes to SHUFFLE (the
// paper's form): gaussblur 1393 vs 1394, gameoflife 1858 vs 1893, jacobi2d9
// 1625 vs 1642, whispering 149 vs 152, divergence 417 vs 422 are SHUFFLE.
static int auto_variant(const stencil_s* h) {
    switch (h->k->kind) {
    case ST_WAVE13PT:      // fp64 512^3: 248 vs 257
    case ST_JACOBI3D7:     // fp32 1024^3: 694 vs 711
    case ST_TRICUBIC:      // fp32 256^3: 166 vs 181
    case ST_TRICUBIC2:     // 166 vs 181
    case ST_UXX1:          // 257 vs 274
        return ST_PLAIN;
    default:               // jacobi2d5 32768^2 2038 vs 1684, lapgsrb 571 vs 517,
        return ST_SHUFFLE; // laplacian 369 vs 360, gradient 325 vs 320, the ties above
    }
}

extern "C" int stencil_set_variant(stencil_t h, int variant) {
    if (!h) return set_error(ST_EARG, "null handle");
    if (variant == ST_AUTO) variant = auto_variant(h);
    if (variant < ST_SHUFFLE || variant > ST_PAPER_UNIFORM)
        return set_error(ST_EUNSUPPORTED, "unknown variant %d", variant);
    if (variant >= ST_PAPER_ORIGINAL && h->k->kind >= ST_TRICUBIC2)
        return set_error(ST_EUNSUPPORTED, "no paper-literal variant for %s (SURVEY §8(f) f3 kinds: SHUFFLE / PLAIN)",
                         h->k->name);
    if (variant >= ST_PAPER_ORIGINAL && h->dtype == ST_F64)
        return set_error(ST_EUNSUPPORTED,
                         "the paper-literal variants cover the fp32/int32 kinds (32-bit shuffles, "
                         "PAPER.md:272-274)");
    if (variant >= ST_PAPER_ORIGINAL && dist_is_p2p(h))
        return set_error(ST_EUNSUPPORTED,
                         "the paper-literal variants have no fused peer-store epilogue: use the NCCL or "
                         "host transport");
    h->variant = variant;
    return ST_OK;
}

extern "C" int stencil_set_fusion(stencil_t h, int sweeps_per_launch) {
    if (!h) return set_error(ST_EARG, "null handle");
    if (sweeps_per_launch < -64 || sweeps_per_launch > 3 || sweeps_per_launch == -1)
        return set_error(ST_EARG, "bad fusion setting %d (0 auto, 1 off, 2 / 3 streaming, -S tile)",
                         sweeps_per_launch);
    if (sweeps_per_launch == 3 && h->k->kind == ST_GAUSSBLUR5X5 && !h->gsep)
        return set_error(ST_EUNSUPPORTED, "gaussblur5x5 with non-separable weights has no three-sweep streaming kernel");
    h->fusion = sweeps_per_launch;
    for (auto& g : h->graphs)          // cached graphs encode the old schedule
        if (g.exec) cudaGraphExecDestroy(g.exec);
    h->graphs.clear();
    return ST_OK;
}

extern "C" int stencil_get_variant(stencil_t h, int* variant) {
    if (!h || !variant) return set_error(ST_EARG, "null argument");
    *variant = h->variant;
    return ST_OK;
}

static int n_bufs_for_run(const KindInfo* k) {
    return k->iterable == 1 ? 2 : k->iterable == 2 ? 3 : k->n_in + k->n_out;
}

extern "C" int stencil_arity(stencil_t h, int* n_in, int* n_out, int* n_bufs) {
    if (!h) return set_error(ST_EARG, "null handle");
    if (n_in) *n_in = h->k->n_in;
    if (n_out) *n_out = h->k->n_out;
    if (n_bufs) *n_bufs = n_bufs_for_run(h->k);
    return ST_OK;
}

int64_t stb200::interior_points(const stencil_s* h) {
    const int lo = h->k->lo, hi = h->k->hi;
    int64_t n = (h->ldims[0] - lo - hi) * (h->ldims[1] - lo - hi);
    if (h->ndims == 3) n *= h->ldims[2] - lo - hi;
    return n;
}

extern "C" int stencil_info(stencil_t h, stencil_info_t* o) {
    if (!h || !o) return set_error(ST_EARG, "null argument");
    memset(o, 0, sizeof *o);
    o->kind = h->k->kind;
    o->dtype = h->dtype;
    o->ndims = h->ndims;
    o->variant = h->variant;
    for (int d = 0; d < 3; ++d) { o->dims[d] = h->dims[d]; o->local_dims[d] = h->ldims[d]; }
    o->lo = h->k->lo;
    o->hi = h->k->hi;
    o->interior_points = interior_points(h);
    if (h->dist) o->interior_points = dist_owned_interior_points(h);
    // compulsory HBM traffic: every input read once, every output written once
    int reads = h->k->n_in, writes = h->k->n_out;
    o->bytes_per_point = (double)(reads + writes) * (double)dtype_size(h->dtype);
    o->launches_per_step = h->dist ? dist_launches_per_step(h) : 1;
    o->sweeps_per_launch = sweeps_per_launch(h, 100);
    o->rank = h->dist ? h->rank : 0;
    o->nranks = h->dist ? h->nranks : 1;
    return ST_OK;
}

extern "C" int stencil_destroy(stencil_t h) {
    if (!h) return ST_OK;
    int dev = -1;
    cudaGetDevice(&dev);
    cudaSetDevice(h->device);
    for (auto& g : h->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
    }
    if (h->cap) cudaStreamDestroy(h->cap);
    if (h->dist) dist_release(h);
    for (auto& tm : h->tmaps) (void)tm;
    if (dev >= 0) cudaSetDevice(dev);
    delete h;
    return ST_OK;
}

// ------------------------------------------------------------ validation
static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static int check_ptrs(const stencil_s* h, const void* const* in, int nin, void* const* out,
                      int nout) {
    if (!in || !out) return set_error(ST_EARG, "null buffer array");
    for (int a = 0; a < nin; ++a) {
        if (!in[a]) return set_error(ST_EARG, "null input %d", a);
        if (!aligned16(in[a])) return set_error(ST_EALIGN, "input %d not 16-byte aligned", a);
    }
    for (int b = 0; b < nout; ++b) {
        if (!out[b]) return set_error(ST_EARG, "null output %d", b);
        if (!aligned16(out[b])) return set_error(ST_EALIGN, "output %d not 16-byte aligned", b);
        for (int a = 0; a < nin; ++a)
            if (out[b] == in[a]) return set_error(ST_EARG, "output %d aliases input %d", b, a);
        for (int c = 0; c < b; ++c)
            if (out[b] == out[c]) return set_error(ST_EARG, "outputs %d and %d alias", b, c);
    }
    (void)h;
    return ST_OK;
}

// ---------------------------------------------------------------- launch
// Enqueue one interior sweep on stream s (no halo exchange).
int stb200::launch_sweep(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                         int64_t z_begin, int64_t z_end) {
    cudaError_t e = dispatch_kernel(h, in, out, s, z_begin, z_end);
    if (e != cudaSuccess)
        return set_error(ST_ECUDA, "%s launch failed: %s", h->k->name, cudaGetErrorString(e));
    return ST_OK;
}

extern "C" int stencil_step(stencil_t h, const void* const* in, void* const* out, void* stream) {
    if (!h) return set_error(ST_EARG, "null handle");
    int rc = check_ptrs(h, in, h->k->n_in, out, h->k->n_out);
    if (rc) return rc;
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (h->dist) return dist_step(h, in, out, s);
    return launch_sweep(h, in, out, s, -1, -1);
}

extern "C" int stencil_step_range(stencil_t h, const void* const* in, void* const* out,
                                  int64_t s_begin, int64_t s_end, void* stream) {
    if (!h) return set_error(ST_EARG, "null handle");
    int rc = check_ptrs(h, in, h->k->n_in, out, h->k->n_out);
    if (rc) return rc;
    const int64_t nslow = h->ldims[h->ndims - 1];
    if (s_begin < h->k->lo || s_end > nslow - h->k->hi || s_begin > s_end)
        return set_error(ST_EARG, "slow-axis range [%lld, %lld) outside the interior [%d, %lld)",
                         (long long)s_begin, (long long)s_end, h->k->lo, (long long)(nslow - h->k->hi));
    cudaSetDevice(h->device);
    if (s_begin == s_end) return ST_OK;
    return launch_sweep(h, in, out, (cudaStream_t)stream, s_begin, s_end);
}

// ------------------------------------------------------ Dirichlet ring copy
// One warp per (k, j) row.  A row is copied whole when it lies in a boundary
// row/plane (slow index outside [full_lo, full_hi), or j outside the
// interior in 3-D); otherwise only its lo + hi edge columns are copied.
template <typename T>
__global__ void __launch_bounds__(128) ring_copy_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                        int64_t nx, int64_t ny, int64_t nz,
                                                        int lo, int hi, int64_t full_lo,
                                                        int64_t full_hi) {
    const int64_t row = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= ny * nz) return;
    const int lane = threadIdx.x & 31;
    const int64_t k = row / ny, j = row % ny;
    const int64_t slow = nz > 1 ? k : j;
    bool full = slow < full_lo || slow >= full_hi;
    if (nz > 1) full = full || j < lo || j >= ny - hi;
    const int64_t base = row * nx;
    if (full) {
        for (int64_t i = lane; i < nx; i += 32) dst[base + i] = src[base + i];
    } else if (lane < lo + hi) {
        const int64_t i = lane < lo ? lane : nx - hi + (lane - lo);
        dst[base + i] = src[base + i];
    }
}

int stb200::ring_copy(const stencil_s* h, const void* src, void* dst, cudaStream_t s) {
    const int64_t nx = h->ldims[0], ny = h->ldims[1], nz = h->ndims == 3 ? h->ldims[2] : 1;
    const int64_t nslow = h->ndims == 3 ? nz : ny;
    int64_t full_lo = h->k->lo, full_hi = nslow - h->k->hi;
    // In a slab decomposition only the global ends own boundary planes; the
    // halo planes of the other ranks are refreshed by the exchange.
    if (h->dist) dist_ring_planes(h, &full_lo, &full_hi);
    const int64_t rows = ny * nz;
    const unsigned blocks = (unsigned)((rows + 3) / 4);
    if (h->dtype == ST_F64)
        ring_copy_kernel<double><<<blocks, 128, 0, s>>>((const double*)src, (double*)dst, nx, ny, nz,
                                                        h->k->lo, h->k->hi, full_lo, full_hi);
    else
        ring_copy_kernel<float><<<blocks, 128, 0, s>>>((const float*)src, (float*)dst, nx, ny, nz,
                                                       h->k->lo, h->k->hi, full_lo, full_hi);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(ST_ECUDA, "ring copy: %s", cudaGetErrorString(e));
    return ST_OK;
}

// ------------------------------------------------------------------ run
// Enqueue the whole run (ring copy + n sweeps) on stream s.  Used both for
// graph capture and (multi-GPU) direct enqueue.
// Sweeps per launch of a 2-D ping-pong run: the handle's fusion setting, or
// (auto) fused when the grid is L2-resident (<= 8 MiB per buffer) and the
// run has several sweeps: there per-launch latency, not HBM, bounds it.
static bool fusable(const stencil_s* h) {
    return h->ndims == 2 && !h->dist && h->k->iterable == 1 && h->variant <= ST_PLAIN;
}
static bool l2_resident(const stencil_s* h) {
    const size_t bytes = (size_t)h->ldims[0] * h->ldims[1] * (h->dtype == ST_F64 ? 8 : 4);
    return bytes <= ((size_t)8 << 20);
}
// Sweeps per launch of the shared-memory tile kernel (ktb2d) for a run, or 1.
static int fusion_depth(const stencil_s* h, int n_iters) {
    if (!fusable(h) || n_iters < 2) return 1;
    const int smax = fused_max_sweeps(h);
    if (h->fusion <= -2) return -h->fusion < smax ? -h->fusion : smax;
    if (h->fusion == 0 && l2_resident(h)) return smax;
    return 1;
}
// Two sweeps per launch through the streaming kernel (k2d2): forced with
// fusion == 2; automatic for jacobi2d5 / jacobi2d9 / gameoflife on grids
// that do not sit in L2.  Measured on B200: jacobi2d5
// 32768^2 fp32 846 -> 1591 Gpt/s, jacobi2d9 846 -> 1622, gameoflife 16384^2
// 832 -> 921, fp64 Jacobi 420 -> ~800; gaussblur (25 FMA/pt, issue-bound
// at two sweeps per pass) is even (805 vs 802) and keeps one sweep per
// launch.
// Sweeps per launch of the streaming kernel for a run (0 = not used).
static int pair_fusion(const stencil_s* h, int n_iters) {
    if (!fusable(h) || n_iters < 2) return 0;
    static const int env_nsw = getenv("STB200_2D_NSW") ? atoi(getenv("STB200_2D_NSW")) : 0;
    const int k = h->k->kind;
    // gaussblur with separable (rank-1) weights: two sweeps per launch
    // (OpGauss5Sep, 10 FMA per point: 8192^2 772 -> 1264 Gpt/s; three run
    // slower, the 25-tap form is issue-bound at two)
    const bool cheap = k == ST_JACOBI2D5 || k == ST_JACOBI2D9 || k == ST_GAMEOFLIFE ||
                       (k == ST_GAUSSBLUR5X5 && h->gsep);
    // three sweeps per launch for jacobi2d5 (measured: 32768^2 fp32 1595 ->
    // 1792 Gpt/s SHUFFLE, fp64 +8%); jacobi2d9 runs slower at three (issue),
    // gaussblur has no three-sweep kernel
    // gameoflife: three with the packed kernel (klife.cuh: 16384^2 1490 -> 1799
    // Gpt/s SHUFFLE, 1505 -> 1862 PLAIN; the int32 form is issue-bound at two)
    static const int life_int = getenv("STB200_LIFE_INT") ? atoi(getenv("STB200_LIFE_INT")) : 0;
    int nsw = k == ST_JACOBI2D5 || (k == ST_GAMEOFLIFE && !life_int) ? 3 : 2;
    if (cheap && env_nsw >= 2 && env_nsw <= 3) nsw = env_nsw;
    if (h->fusion == 2 || h->fusion == 3) nsw = h->fusion;   // forced: exactly that many
    if (nsw > n_iters) nsw = n_iters;
    if (h->fusion == 2 || h->fusion == 3) return nsw;
    return h->fusion == 0 && cheap && !l2_resident(h) ? nsw : 0;
}
int stb200::sweeps_per_launch(const stencil_s* h, int n_iters) {
    const int nsw = pair_fusion(h, n_iters);
    return nsw ? nsw : fusion_depth(h, n_iters);
}

static int enqueue_run(stencil_s* h, void* const* bufs, int n_iters, cudaStream_t s, int* result) {
    const KindInfo* k = h->k;
    int rc;
    if (dist_is_p2p(h)) return p2p_run(h, bufs, n_iters, s, result);
    if (k->iterable == 1) {
        if (const int nsw = pair_fusion(h, n_iters)) {
            // nsw sweeps per launch (k2d2); a remainder runs first as single
            // sweeps.  The ring stays fixed: copy it once, as below.
            if ((rc = ring_copy(h, bufs[0], bufs[1], s))) return rc;
            int cur = 0, done = 0;
            for (; done < n_iters % nsw; ++done) {
                const void* in[1] = {bufs[cur]};
                void* out[1] = {bufs[1 - cur]};
                if ((rc = launch_sweep(h, in, out, s, -1, -1))) return rc;
                cur = 1 - cur;
            }
            for (; done < n_iters; done += nsw) {
                cudaError_t e = dispatch_2d_pair(h, bufs[cur], bufs[1 - cur], s, nsw);
                if (e != cudaSuccess)
                    return set_error(ST_ECUDA, "%s two-sweep launch failed: %s", k->name, cudaGetErrorString(e));
                cur = 1 - cur;
            }
            *result = cur;
            return ST_OK;
        }
        const int S = fusion_depth(h, n_iters);
        if (S > 1) {
            // as few passes of <= S sweeps as possible (one launch for a run
            // of up to S sweeps; the fused kernels also write the ring cells,
            // so no ring copy); the result buffer is reported in *result
            const int passes = (n_iters + S - 1) / S;
            int cur = 0, done = 0;
            for (int p = 0; p < passes; ++p) {
                const int sw = (n_iters - done) / (passes - p);     // even split, each >= 1
                cudaError_t e = dispatch_2d_fused(h, bufs[cur], bufs[1 - cur], s, sw);
                if (e != cudaSuccess)
                    return set_error(ST_ECUDA, "%s fused launch failed: %s", k->name, cudaGetErrorString(e));
                done += sw;
                cur = 1 - cur;
            }
            *result = cur;
            return ST_OK;
        }
        if ((rc = ring_copy(h, bufs[0], bufs[1], s))) return rc;
        int cur = 0;
        for (int it = 0; it < n_iters; ++it) {
            const void* in[1] = {bufs[cur]};
            void* out[1] = {bufs[1 - cur]};
            rc = h->dist ? dist_step(h, in, out, s) : launch_sweep(h, in, out, s, -1, -1);
            if (rc) return rc;
            cur = 1 - cur;
        }
        *result = cur;
        return ST_OK;
    }
    if (k->iterable == 2) {
        if ((rc = ring_copy(h, bufs[1], bufs[0], s))) return rc;
        if ((rc = ring_copy(h, bufs[1], bufs[2], s))) return rc;
        int p = 0, c = 1, n = 2;
        for (int it = 0; it < n_iters; ++it) {
            const void* in[2] = {bufs[p], bufs[c]};
            void* out[1] = {bufs[n]};
            rc = h->dist ? dist_step(h, in, out, s) : launch_sweep(h, in, out, s, -1, -1);
            if (rc) return rc;
            const int t = p; p = c; c = n; n = t;
        }
        *result = c;
        return ST_OK;
    }
    const void* in[8];
    void* out[3];
    for (int a = 0; a < k->n_in; ++a) in[a] = bufs[a];
    for (int b = 0; b < k->n_out; ++b) out[b] = bufs[k->n_in + b];
    for (int it = 0; it < n_iters; ++it) {
        rc = h->dist ? dist_step(h, in, out, s) : launch_sweep(h, in, out, s, -1, -1);
        if (rc) return rc;
    }
    *result = k->n_in;
    return ST_OK;
}

extern "C" int stencil_run(stencil_t h, void* const* bufs, int n_iters, void* stream,
                           int* result_idx) {
    if (!h || !bufs) return set_error(ST_EARG, "null argument");
    if (n_iters < 0) return set_error(ST_EARG, "n_iters < 0");
    const int nb = n_bufs_for_run(h->k);
    for (int a = 0; a < nb; ++a) {
        if (!bufs[a]) return set_error(ST_EARG, "null buffer %d", a);
        if (!aligned16(bufs[a])) return set_error(ST_EALIGN, "buffer %d not 16-byte aligned", a);
        for (int b = 0; b < a; ++b)
            if (bufs[a] == bufs[b]) return set_error(ST_EARG, "buffers %d and %d alias", a, b);
    }
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    int result = 0;

    // Multi-GPU runs are enqueued directly: the NCCL calls inside each step
    // are issued on a side stream with events (see dist.cu).  So is a run
    // that is ONE kernel launch (all sweeps of a small 2-D run in ktb2r,
    // no ring copy): a graph would only add its launch latency.
    const bool one_launch = h->k->iterable == 1 && n_iters >= 1 && !pair_fusion(h, n_iters) &&
                            fusion_depth(h, n_iters) >= n_iters;
    if (h->dist || one_launch) {
        int rc = enqueue_run(h, bufs, n_iters, s, &result);
        if (!rc && result_idx) *result_idx = result;
        return rc;
    }

    // Single GPU: one cached CUDA graph per (bufs, n_iters, variant).
    GraphEntry* hit = nullptr;
    for (auto& g : h->graphs) {
        bool same = g.n_iters == n_iters && g.variant == h->variant && g.nb == nb;
        for (int a = 0; same && a < nb; ++a) same = g.bufs[a] == bufs[a];
        if (same) { hit = &g; break; }
    }
    if (!hit) {
        if (!h->cap) {
            cudaError_t e = cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking);
            if (e != cudaSuccess) return set_error(ST_ECUDA, "stream create: %s", cudaGetErrorString(e));
        }
        if (h->graphs.size() >= 8) {
            cudaGraphExecDestroy(h->graphs.front().exec);
            h->graphs.erase(h->graphs.begin());
        }
        GraphEntry g{};
        g.n_iters = n_iters;
        g.variant = h->variant;
        g.nb = nb;
        for (int a = 0; a < nb; ++a) g.bufs[a] = bufs[a];
        cudaError_t e = cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return set_error(ST_ECUDA, "begin capture: %s", cudaGetErrorString(e));
        int rc = enqueue_run(h, bufs, n_iters, h->cap, &g.result);
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(h->cap, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return set_error(ST_ECUDA, "end capture: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return set_error(ST_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
        h->graphs.push_back(g);
        hit = &h->graphs.back();
    }
    cudaError_t e = cudaGraphLaunch(hit->exec, s);
    if (e != cudaSuccess) return set_error(ST_ECUDA, "graph launch: %s", cudaGetErrorString(e));
    if (result_idx) *result_idx = hit->result;
    return ST_OK;
}

extern "C" int stencil_run_host_async(stencil_t h, const void* const* host_in, void* const* host_out,
                                      void* const* dev_bufs, int n_iters, void* stream) {
    if (!h || !host_in || !host_out || !dev_bufs) return set_error(ST_EARG, "null argument");
    cudaSetDevice(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    const KindInfo* k = h->k;
    const size_t bytes = (size_t)h->ldims[0] * h->ldims[1] * h->ldims[2] * dtype_size(h->dtype);
    // inputs -> their run-buffer slots
    const int n_up = k->iterable == 1 ? 1 : k->iterable == 2 ? 2 : k->n_in;
    for (int a = 0; a < n_up; ++a) {
        cudaError_t e = cudaMemcpyAsync(dev_bufs[a], host_in[a], bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return set_error(ST_ECUDA, "H2D copy: %s", cudaGetErrorString(e));
    }
    int result = 0;
    int rc = stencil_run(h, dev_bufs, n_iters, stream, &result);
    if (rc) return rc;
    const int n_down = k->iterable ? 1 : k->n_out;
    for (int b = 0; b < n_down; ++b) {
        cudaError_t e = cudaMemcpyAsync(host_out[b], dev_bufs[result + b], bytes,
                                        cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return set_error(ST_ECUDA, "D2H copy: %s", cudaGetErrorString(e));
    }
    return ST_OK;
}

extern "C" int stencil_run_host(stencil_t h, const void* const* host_in, void* const* host_out,
                                void* const* dev_bufs, int n_iters, void* stream) {
    const int rc = stencil_run_host_async(h, host_in, host_out, dev_bufs, n_iters, stream);
    if (rc) return rc;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return set_error(ST_ECUDA, "sync: %s", cudaGetErrorString(e));
    return ST_OK;
}
