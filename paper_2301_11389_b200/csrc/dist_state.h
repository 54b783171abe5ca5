// dist_state.h — multi-GPU state shared by dist.cu (NCCL / host transports)
// and p2p.cu (fused peer-store transport).  Not part of the C ABI.
#pragma once
#include <vector>

#include "internal.h"

// Minimal NCCL ABI subset (nccl.h, NCCL 2.x; stable since 2.0).
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;                       // ncclSuccess = 0
typedef struct { char internal[128]; } ncclUniqueId;
static const int kNcclInt8 = 0;                 // ncclInt8 == ncclChar

namespace stb200 {

struct P2PState;                   // p2p.cu

struct DistState {
    // transport: NCCL (default) or a host callback (stencil_dist_attach_host)
    stencil_exchange_fn host_fn = nullptr;
    void* host_user = nullptr;
    char* host_buf = nullptr;        // pinned staging: send lo | send hi | recv lo | recv hi
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t e_in = nullptr, e_comm = nullptr;
    int64_t n = 0, m = 0;            // global slow extent, planes per rank
    int64_t plan[8] = {0};
    size_t plane_bytes = 0;
    P2PState* p2p = nullptr;         // fused peer-store transport (p2p.cu), else null
};

// p2p.cu
int p2p_step(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s);
int p2p_run(stencil_s* h, void* const* bufs, int n_iters, cudaStream_t s, int* result);
void p2p_release(DistState* d);
// dist.cu helpers used by p2p.cu
void dist_output_slabs(const stencil_s* h, int64_t* a, int64_t* x0, int64_t* x1, int64_t* b);
unsigned dist_halo_inputs(int kind);
}  // namespace stb200
int dist_attach_common(stencil_t h, int rank, int nranks, stb200::DistState** out);
void dist_attach_finish(stencil_t h, stb200::DistState* d, int rank, int nranks);
