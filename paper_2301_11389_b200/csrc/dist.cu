// dist.cu — 1-D slab decomposition along the slowest axis with NCCL halo
// exchange over NVLink / NVSwitch, one process per GPU.
//
// Not in the paper (single GPU): the decomposition named by
// BASELINE.json north_star.  Layout: the global slow extent n (boundary
// planes included) is split into N slabs of m = n/N planes; every rank's
// local buffers hold lo + m + hi planes, local plane L <-> global plane
// p*m - lo + L.  Rank 0's first lo and rank N-1's last hi local planes lie
// outside the domain and are never read.
//
// One step (stencil_step) on rank p:
//   s:    record e_in                         (inputs of this step complete)
//   comm: wait e_in; ncclGroupStart;
//           send local [lo, lo+hi)  -> p-1;  recv local [0, lo)        <- p-1
//           send local [m, m+lo)    -> p+1;  recv local [lo+m, lo+m+hi) <- p+1
//         ncclGroupEnd; record e_comm
//   s:    interior kernel over the output planes that read no halo plane
//         (overlaps the exchange), wait e_comm, then the (at most two) thin
//         slabs of output planes that read a halo plane.
// Results are bit-identical to one GPU: per-point arithmetic is unchanged.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include "internal.h"
#include "dist_state.h"

namespace stb200 {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// The process's libnccl.so.2 (the one torch already loaded, if any: dlopen
// returns the resident copy, so only one NCCL lives in the process).
static NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (so) {
#define LOAD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(so, "nccl" #f))
            LOAD(GetUniqueId); LOAD(CommInitRank); LOAD(CommDestroy); LOAD(Send); LOAD(Recv);
            LOAD(GroupStart); LOAD(GroupEnd); LOAD(GetErrorString);
#undef LOAD
            api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send &&
                     api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
        }
    }
    return api;
}

// Inputs with taps along the slow axis (their halo planes must be exchanged).
static unsigned halo_inputs(int kind) {
    switch (kind) {
    case ST_WAVE13PT: return 1u << 1;      // cur; prev is read at the centre only
    case ST_DIVERGENCE: return 1u << 2;    // w carries the z taps
    default: return 1u;                    // the single field / u / f
    }
}

int64_t dist_owned_interior_points(const stencil_s* h) {
    const DistState* d = h->dist;
    const int lo = h->k->lo, hi = h->k->hi;
    const int64_t ga = std::max<int64_t>((int64_t)h->rank * d->m, lo);
    const int64_t gb = std::min<int64_t>((int64_t)(h->rank + 1) * d->m, d->n - hi);
    int64_t planes = gb > ga ? gb - ga : 0;
    int64_t per = h->ldims[0] - lo - hi;
    if (h->ndims == 3) per *= h->ldims[1] - lo - hi;
    return planes * per;
}

// Output slabs of this rank in local planes: [a, b) owned interior, split into
// lower halo-dependent [a, x0), independent [x0, x1), upper dependent [x1, b).
static void output_slabs(const stencil_s* h, int64_t* a, int64_t* x0, int64_t* x1, int64_t* b) {
    const DistState* d = h->dist;
    const int lo = h->k->lo, hi = h->k->hi;
    const int64_t base = (int64_t)h->rank * d->m;
    const int64_t ga = std::max<int64_t>(base, lo), gb = std::min<int64_t>(base + d->m, d->n - hi);
    *a = ga - base + lo;
    *b = gb - base + lo;
    if (*b < *a) *b = *a;
    const bool has_lower = h->rank > 0, has_upper = h->rank < h->nranks - 1;
    int64_t dep_lo_end = has_lower ? 2 * lo : *a;          // outputs < 2lo read planes < lo
    int64_t dep_hi_begin = has_upper ? lo + d->m - hi : *b; // outputs >= lo+m-hi read >= lo+m
    *x0 = std::min(std::max(*a, dep_lo_end), *b);
    *x1 = std::max(std::min(*b, dep_hi_begin), *x0);
}

int dist_launches_per_step(const stencil_s* h) {
    int64_t a, x0, x1, b;
    output_slabs(h, &a, &x0, &x1, &b);
    if (h->dist->p2p) return b > a;    // one launch with fused peer stores
    return (x0 > a) + (x1 > x0) + (b > x1);
}

static int nccl_check(ncclResult_t r, const char* what) {
    if (r == 0) return ST_OK;
    return set_error(ST_ENCCL, "%s: %s", what, nccl().GetErrorString(r));
}

// Host transport (test / no-NCCL deployments): synchronous, no overlap.
static int host_exchange(stencil_s* h, const void* const* in, cudaStream_t s) {
    DistState* d = h->dist;
    const size_t pb = d->plane_bytes;
    const int64_t recv_lo_at = d->plan[3], send_lo_from = d->plan[4];
    const int64_t recv_hi_at = d->plan[5], send_hi_from = d->plan[6];
    const size_t n_lo = (size_t)(d->plan[7] & 0xFFFF), n_hi = (size_t)(d->plan[7] >> 16);
    const unsigned mask = halo_inputs(h->k->kind);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_error(ST_ECUDA, "sync: %s", cudaGetErrorString(e));
    for (int a = 0; a < h->k->n_in; ++a) {
        if (!(mask >> a & 1u)) continue;
        char* buf = (char*)in[a];
        if (h->rank > 0) {
            // staging layout: send-lo [0, n_hi) | send-hi [n_hi, n_hi+n_lo) |
            // recv-lo [n_hi+n_lo, n_hi+2n_lo) | recv-hi [n_hi+2n_lo, 2n_hi+2n_lo) planes
            char* snd = d->host_buf;
            char* rcv = d->host_buf + (n_hi + n_lo) * pb;
            cudaMemcpy(snd, buf + (size_t)send_lo_from * pb, n_hi * pb, cudaMemcpyDeviceToHost);
            if (d->host_fn(h->rank - 1, snd, n_hi * pb, rcv, n_lo * pb, d->host_user))
                return set_error(ST_ENCCL, "host exchange with rank %d failed", h->rank - 1);
            cudaMemcpy(buf + (size_t)recv_lo_at * pb, rcv, n_lo * pb, cudaMemcpyHostToDevice);
        }
        if (h->rank < h->nranks - 1) {
            char* snd = d->host_buf + n_hi * pb;
            char* rcv = d->host_buf + (n_hi + 2 * n_lo) * pb;
            cudaMemcpy(snd, buf + (size_t)send_hi_from * pb, n_lo * pb, cudaMemcpyDeviceToHost);
            if (d->host_fn(h->rank + 1, snd, n_lo * pb, rcv, n_hi * pb, d->host_user))
                return set_error(ST_ENCCL, "host exchange with rank %d failed", h->rank + 1);
            cudaMemcpy(buf + (size_t)recv_hi_at * pb, rcv, n_hi * pb, cudaMemcpyHostToDevice);
        }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(ST_ECUDA, "host exchange copy: %s", cudaGetErrorString(e));
    return ST_OK;
}

bool dist_is_p2p(const stencil_s* h) { return h->dist && h->dist->p2p; }

void dist_output_slabs(const stencil_s* h, int64_t* a, int64_t* x0, int64_t* x1, int64_t* b) {
    output_slabs(h, a, x0, x1, b);
}
unsigned dist_halo_inputs(int kind) { return halo_inputs(kind); }

int dist_step(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s) {
    DistState* d = h->dist;
    if (d->p2p) return p2p_step(h, in, out, s);
    int rc;
    int64_t a, x0, x1, b;
    output_slabs(h, &a, &x0, &x1, &b);
    if (d->host_fn) {                  // host transport: exchange, then all slabs
        if ((rc = host_exchange(h, in, s))) return rc;
        if (x0 > a && (rc = launch_sweep(h, in, out, s, a, x0))) return rc;
        if (x1 > x0 && (rc = launch_sweep(h, in, out, s, x0, x1))) return rc;
        if (b > x1 && (rc = launch_sweep(h, in, out, s, x1, b))) return rc;
        return ST_OK;
    }
    NcclApi& api = nccl();
    const size_t pb = d->plane_bytes;
    const bool has_lower = h->rank > 0, has_upper = h->rank < h->nranks - 1;
    cudaError_t e;

    // 1. exchange the halo planes of every input with slow-axis taps
    if ((e = cudaEventRecord(d->e_in, s)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(d->comm_stream, d->e_in, 0)) != cudaSuccess)
        return set_error(ST_ECUDA, "event: %s", cudaGetErrorString(e));
    if ((rc = nccl_check(api.GroupStart(), "ncclGroupStart"))) return rc;
    const unsigned mask = halo_inputs(h->k->kind);
    // offsets and counts straight from the host plan (stencil_slab_plan)
    const int64_t recv_lo_at = d->plan[3], send_lo_from = d->plan[4];
    const int64_t recv_hi_at = d->plan[5], send_hi_from = d->plan[6];
    const size_t n_lo = (size_t)(d->plan[7] & 0xFFFF), n_hi = (size_t)(d->plan[7] >> 16);
    // a failed enqueue still closes the group (NCCL requires balanced
    // GroupStart / GroupEnd) before the first error is returned
    int first = ST_OK;
    auto chk = [&](ncclResult_t r, const char* what) {
        if (r != 0 && first == ST_OK) first = nccl_check(r, what);
    };
    for (int ai = 0; ai < h->k->n_in; ++ai) {
        if (!(mask >> ai & 1u)) continue;
        char* buf = (char*)in[ai];     // the halo planes of an input are the exchange's
        if (has_lower) {               // my bottom hi owned planes <-> rank-1's top lo planes
            chk(api.Send(buf + (size_t)send_lo_from * pb, n_hi * pb, kNcclInt8, h->rank - 1, d->comm,
                         d->comm_stream), "ncclSend to rank-1");
            chk(api.Recv(buf + (size_t)recv_lo_at * pb, n_lo * pb, kNcclInt8, h->rank - 1, d->comm,
                         d->comm_stream), "ncclRecv from rank-1");
        }
        if (has_upper) {               // my top lo owned planes <-> rank+1's bottom hi planes
            chk(api.Send(buf + (size_t)send_hi_from * pb, n_lo * pb, kNcclInt8, h->rank + 1, d->comm,
                         d->comm_stream), "ncclSend to rank+1");
            chk(api.Recv(buf + (size_t)recv_hi_at * pb, n_hi * pb, kNcclInt8, h->rank + 1, d->comm,
                         d->comm_stream), "ncclRecv from rank+1");
        }
    }
    rc = nccl_check(api.GroupEnd(), "ncclGroupEnd");
    if (first) return first;
    if (rc) return rc;
    if ((e = cudaEventRecord(d->e_comm, d->comm_stream)) != cudaSuccess)
        return set_error(ST_ECUDA, "event: %s", cudaGetErrorString(e));

    // 2. interior planes (overlap the exchange), 3. halo-dependent slabs
    if (x1 > x0 && (rc = launch_sweep(h, in, out, s, x0, x1))) return rc;
    if ((e = cudaStreamWaitEvent(s, d->e_comm, 0)) != cudaSuccess)
        return set_error(ST_ECUDA, "event wait: %s", cudaGetErrorString(e));
    if (x0 > a && (rc = launch_sweep(h, in, out, s, a, x0))) return rc;
    if (b > x1 && (rc = launch_sweep(h, in, out, s, x1, b))) return rc;
    return ST_OK;
}

void dist_release(stencil_s* h) {
    DistState* d = h->dist;
    if (!d) return;
    if (d->comm && nccl().ok) nccl().CommDestroy(d->comm);
    if (d->host_buf) cudaFreeHost(d->host_buf);
    if (d->p2p) p2p_release(d);
    if (d->e_in) cudaEventDestroy(d->e_in);
    if (d->e_comm) cudaEventDestroy(d->e_comm);
    if (d->comm_stream) cudaStreamDestroy(d->comm_stream);
    delete d;
    h->dist = nullptr;
}

// Full-plane ranges of the Dirichlet ring copy in local slow-axis planes.
void dist_ring_planes(const stencil_s* h, int64_t* full_lo, int64_t* full_hi) {
    // local plane L holds global plane rank*m - lo + L; global planes < lo and
    // >= n - hi are the Dirichlet boundary.  They are copied whole: rank 0's
    // dead + boundary planes, the last rank's, and (slabs thinner than 2*lo
    // or 2*hi) boundary planes that sit in a middle rank's halo, which no
    // rank computes and the fused peer stores therefore never refresh.
    const int lo = h->k->lo, hi = h->k->hi;
    const int64_t m = h->dist->m, base = (int64_t)h->rank * m;
    *full_lo = std::max<int64_t>(0, 2 * lo - base);
    *full_hi = std::min<int64_t>(lo + m + hi, h->dist->n - hi - base + lo);
}

}  // namespace stb200

using namespace stb200;

extern "C" int stencil_slab_plan(int64_t n, int lo, int hi, int rank, int nranks, int64_t plan[8]) {
    if (!plan) return set_error(ST_EARG, "null plan");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(ST_EARG, "bad rank/nranks");
    if (lo < 0 || hi < 0 || lo > 0xFFFF || hi > 0xFFFF) return set_error(ST_EARG, "bad halo");
    if (n % nranks) return set_error(ST_EARG, "slow extent %lld not divisible by %d", (long long)n, nranks);
    const int64_t m = n / nranks;
    if (m < lo || m < hi || m < 1) return set_error(ST_EARG, "slab of %lld planes thinner than the halo", (long long)m);
    plan[0] = (int64_t)rank * m;                    // own_begin (global)
    plan[1] = (int64_t)(rank + 1) * m;              // own_end (global)
    plan[2] = m + lo + hi;                          // local planes
    plan[3] = rank > 0 ? 0 : -1;                    // recv_lo_at   (lo planes from rank-1)
    plan[4] = rank > 0 ? lo : -1;                   // send_lo_from (hi planes to rank-1)
    plan[5] = rank < nranks - 1 ? lo + m : -1;      // recv_hi_at   (hi planes from rank+1)
    plan[6] = rank < nranks - 1 ? m : -1;           // send_hi_from (lo planes to rank+1)
    plan[7] = (int64_t)lo | ((int64_t)hi << 16);
    return ST_OK;
}

extern "C" int stencil_dist_get_id(uint8_t id[128]) {
    if (!id) return set_error(ST_EARG, "null id");
    NcclApi& api = nccl();
    if (!api.ok) return set_error(ST_ENCCL, "libnccl.so.2 not loadable: %s", dlerror());
    ncclUniqueId u;
    int rc = nccl_check(api.GetUniqueId(&u), "ncclGetUniqueId");
    if (rc) return rc;
    memcpy(id, u.internal, 128);
    return ST_OK;
}

// Common part of attaching: plan, streams/events, local dims.
int dist_attach_common(stencil_t h, int rank, int nranks, DistState** out) {
    if (!h) return set_error(ST_EARG, "null handle");
    if (h->dist) return set_error(ST_ESTATE, "handle already attached");
    if (!h->graphs.empty()) return set_error(ST_ESTATE, "attach before the first run");
    if (h->k->kind >= ST_TRICUBIC2)
        return set_error(ST_EUNSUPPORTED, "%s runs on one GPU (SURVEY §8(f) f3 kind: no slab decomposition)",
                         h->k->name);
    const int slow = h->ndims - 1;
    int64_t plan[8];
    int rc = stencil_slab_plan(h->dims[slow], h->k->lo, h->k->hi, rank, nranks, plan);
    if (rc) return rc;
    cudaSetDevice(h->device);
    DistState* d = new DistState();
    d->n = h->dims[slow];
    d->m = d->n / nranks;
    memcpy(d->plan, plan, sizeof plan);
    const size_t es = h->dtype == ST_F64 ? 8 : 4;
    d->plane_bytes = (size_t)h->dims[0] * (h->ndims == 3 ? (size_t)h->dims[1] : 1) * es;
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&d->comm_stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&d->e_in, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&d->e_comm, cudaEventDisableTiming)) != cudaSuccess) {
        h->dist = d;
        dist_release(h);
        return set_error(ST_ECUDA, "attach: %s", cudaGetErrorString(e));
    }
    *out = d;
    return ST_OK;
}

void dist_attach_finish(stencil_t h, DistState* d, int rank, int nranks) {
    h->dist = d;
    h->rank = rank;
    h->nranks = nranks;
    h->ldims[h->ndims - 1] = d->plan[2];
}

extern "C" int stencil_dist_attach(stencil_t h, const uint8_t id[128], int rank, int nranks) {
    if (!id) return set_error(ST_EARG, "null id");
    NcclApi& api = nccl();
    if (!api.ok) return set_error(ST_ENCCL, "libnccl.so.2 not loadable");
    DistState* d = nullptr;
    int rc = dist_attach_common(h, rank, nranks, &d);
    if (rc) return rc;
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    rc = nccl_check(api.CommInitRank(&d->comm, nranks, u, rank), "ncclCommInitRank");
    if (rc) {
        d->comm = nullptr;
        h->dist = d;
        dist_release(h);
        return rc;
    }
    dist_attach_finish(h, d, rank, nranks);
    return ST_OK;
}

extern "C" int stencil_dist_attach_host(stencil_t h, int rank, int nranks, stencil_exchange_fn fn,
                                        void* user) {
    if (!fn) return set_error(ST_EARG, "null exchange function");
    DistState* d = nullptr;
    int rc = dist_attach_common(h, rank, nranks, &d);
    if (rc) return rc;
    const size_t n_lo = (size_t)(d->plan[7] & 0xFFFF), n_hi = (size_t)(d->plan[7] >> 16);
    cudaError_t e = cudaMallocHost(&d->host_buf, 2 * (n_lo + n_hi) * d->plane_bytes);
    if (e != cudaSuccess) {
        h->dist = d;
        dist_release(h);
        return set_error(ST_ECUDA, "pinned staging: %s", cudaGetErrorString(e));
    }
    d->host_fn = fn;
    d->host_user = user;
    dist_attach_finish(h, d, rank, nranks);
    return ST_OK;
}
