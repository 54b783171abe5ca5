// internal.h — handle layout and cross-file declarations of libstencil_b200
// (not part of the C ABI).
#pragma once
#include <cstdarg>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/stencil.h"

namespace stb200 {

struct KindInfo {
    int kind;
    const char* name;
    int ndims, n_in, n_out, lo, hi, ncoeffs;
    int iterable;          // 1 ping-pong, 2 three-level (wave13pt), 0 re-apply
    bool allow_f, allow_i;
};

struct GraphEntry {
    void* bufs[16];
    int nb, n_iters, variant, result;
    cudaGraphExec_t exec;
};

struct DistState;          // dist.cu

}  // namespace stb200

struct stencil_s {
    const stb200::KindInfo* k = nullptr;
    int dtype = 0, ndims = 0, variant = 0, device = 0;
    int fusion = 0;                  // 0 auto, 1 off, >= 2 sweeps per launch (2-D run)
    int64_t dims[3] = {1, 1, 1};     // global
    int64_t ldims[3] = {1, 1, 1};    // local buffers (slab + halo when attached)
    double coeffs[32] = {0};
    cudaStream_t cap = nullptr;      // graph-capture stream
    std::vector<stb200::GraphEntry> graphs;
    std::vector<int> tmaps;          // reserved
    // multi-GPU
    stb200::DistState* dist = nullptr;
    // fused halo stores for the next launch (dist.cu P2P transport; null = off)
    void* peer_lo = nullptr;
    void* peer_hi = nullptr;
    int64_t peer_lo_end = 0, peer_hi_begin = 0, peer_d_lo = 0, peer_d_hi = 0;
    int rank = 0, nranks = 1;
    // gaussblur5x5 weights factored as w[dj][di] = u[dj] * v[di] (api.cu, at
    // create): the separable kernels' coefficients (u[0..4], v[0..4])
    bool gsep = false;
    double gsep_c[10] = {0};
};

namespace stb200 {

int set_error(int code, const char* fmt, ...);
// Per (kernel, device) one-time setup, thread-safe: opts the kernel in to
// `smem` bytes of dynamic shared memory on `device` (the attribute is per
// device context, so a handle on a second GPU needs its own call) and
// returns its resident blocks per SM at (threads, smem), >= 1.  A later
// call with a larger smem re-applies the attribute.  api.cu.
int kernel_setup(const void* func, int device, size_t smem, int threads);
const KindInfo* kind_info(int kind);
int64_t interior_points(const stencil_s* h);

// Launch the kernel of h for output slow-axis range [s_begin, s_end) of the
// local buffers (-1,-1 = the whole interior).  dispatch.cu.
cudaError_t dispatch_kernel(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                            int64_t s_begin, int64_t s_end);
int launch_sweep(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                 int64_t s_begin, int64_t s_end);
// dispatch2d.cu: temporally blocked 2-D sweeps
cudaError_t dispatch_2d_fused(stencil_s* h, const void* in, void* out, cudaStream_t s, int S);
int fused_max_sweeps(const stencil_s* h);
cudaError_t dispatch_2d_pair(stencil_s* h, const void* in, void* out, cudaStream_t s, int nsw);
int sweeps_per_launch(const stencil_s* h, int n_iters);
int ring_copy(const stencil_s* h, const void* src, void* dst, cudaStream_t s);

// dist.cu
int dist_step(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s);
void dist_release(stencil_s* h);
int64_t dist_owned_interior_points(const stencil_s* h);
int dist_launches_per_step(const stencil_s* h);
void dist_ring_planes(const stencil_s* h, int64_t* full_lo, int64_t* full_hi);
bool dist_is_p2p(const stencil_s* h);
int p2p_run(stencil_s* h, void* const* bufs, int n_iters, cudaStream_t s, int* result);

}  // namespace stb200
