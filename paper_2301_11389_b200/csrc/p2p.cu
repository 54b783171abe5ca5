// p2p.cu — fused halo exchange over peer memory (multi-GPU, one process per
// GPU): the compute kernel that produces a rank's boundary planes also stores
// them straight into the neighbours' buffers through CUDA-IPC peer pointers
// (P2P over NVLink / NVSwitch; two processes on one GPU in the tests), so the
// transfer overlaps the math plane by plane and no copy or collective kernel
// runs.  Ordering between ranks uses epoch flags in device memory written
// and waited on by stream memory operations (cuStreamWriteValue32 /
// cuStreamWaitValue32: the wait happens in the GPU front end, no SM spins):
//
//   flags[0] = done        last epoch whose input this rank finished reading
//   flags[1] = ready_lo    halos from rank-1 are in place for this epoch
//   flags[2] = ready_hi    halos from rank+1 are in place for this epoch
//
// A run on rank p (epoch e0 before it):
//   prologue  wait done[q] >= e0; copy my boundary planes of the current field
//             into q's halo planes (peer copy); ready[q] = e0+1
//   step e    wait ready_lo/hi >= e;  wait done[q] >= e-1 (q's buffer free);
//             launches with fused peer stores of the output's boundary planes;
//             ready[q] = e+1; done = e
// Non-iterable kinds (static inputs) exchange their input halos once.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/stencil.h"
#include "dist_state.h"
#include "internal.h"

namespace stb200 {

struct PeerSet {                       // one registered buffer set of a run
    int nb = 0;
    void* local[8] = {};
    char* peer[2][8] = {};             // [0] lower neighbour, [1] upper neighbour
};

struct P2PState {
    uint32_t* flags = nullptr;         // mine: done, ready_lo, ready_hi
    uint32_t* pflags[2] = {nullptr, nullptr};
    uint32_t epoch = 0;
    unsigned wait_flags = CU_STREAM_WAIT_VALUE_GEQ;   // | FLUSH where the device supports it
    std::vector<PeerSet> sets;
    std::map<std::string, char*> opened;   // IPC handle bytes -> mapped base
};

struct DrvApi {
    PFN_cuStreamWaitValue32_v11070 wait = nullptr;
    PFN_cuStreamWriteValue32_v11070 write = nullptr;
    PFN_cuMemGetAddressRange_v3020 range = nullptr;
    bool ok = false;
};

static DrvApi& drv() {
    static DrvApi a;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            a.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            a.write = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            a.range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
        a.ok = a.wait && a.write && a.range;
    }
    return a;
}

// flags: CU_STREAM_WAIT_VALUE_GEQ, plus CU_STREAM_WAIT_VALUE_FLUSH (flush the
// remote writes that arrived before the flag) where the device supports it.
static int wait_geq(cudaStream_t s, const uint32_t* addr, uint32_t v,
                    unsigned flags = CU_STREAM_WAIT_VALUE_GEQ) {
    CUresult r = drv().wait((CUstream)s, (CUdeviceptr)addr, v, flags);
    return r == CUDA_SUCCESS ? ST_OK : set_error(ST_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
}
static int write_val(cudaStream_t s, uint32_t* addr, uint32_t v) {
    CUresult r = drv().write((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT);
    return r == CUDA_SUCCESS ? ST_OK : set_error(ST_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
}

void p2p_release(DistState* d) {
    P2PState* p = d->p2p;
    if (!p) return;
    for (auto& kv : p->opened) cudaIpcCloseMemHandle(kv.second);
    if (p->flags) cudaFree(p->flags);
    delete p;
    d->p2p = nullptr;
}

static const PeerSet* find_set(const P2PState* p, const void* buf, int* idx) {
    for (const auto& ps : p->sets)
        for (int k = 0; k < ps.nb; ++k)
            if (ps.local[k] == buf) {
                *idx = k;
                return &ps;
            }
    return nullptr;
}

// Copy my boundary planes of buffer k of set ps into the neighbours' halo
// planes once they are done with epoch `wait_done`, signal ready = `sig`,
// then wait until my own halos are signalled `sig`.
static int exchange_inputs(stencil_s* h, const PeerSet* ps, int k, cudaStream_t s, uint32_t wait_done,
                           uint32_t sig) {
    DistState* d = h->dist;
    P2PState* p = d->p2p;
    const size_t pb = d->plane_bytes;
    const int64_t m = d->m;
    const int lo = h->k->lo, hi = h->k->hi;
    const bool has[2] = {h->rank > 0, h->rank < h->nranks - 1};
    int rc;
    char* mine = (char*)ps->local[k];
    for (int q = 0; q < 2; ++q) {
        if (!has[q]) continue;
        if ((rc = wait_geq(s, p->pflags[q], wait_done))) return rc;
        cudaError_t e;
        if (q == 0)   // lower neighbour's upper halo [lo+m, lo+m+hi) <- my planes [lo, lo+hi)
            e = cudaMemcpyAsync(ps->peer[0][k] + (size_t)(lo + m) * pb, mine + (size_t)lo * pb, (size_t)hi * pb,
                                cudaMemcpyDeviceToDevice, s);
        else          // upper neighbour's lower halo [0, lo) <- my planes [m, m+lo)
            e = cudaMemcpyAsync(ps->peer[1][k], mine + (size_t)m * pb, (size_t)lo * pb,
                                cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return set_error(ST_ECUDA, "peer copy: %s", cudaGetErrorString(e));
        // I am q's upper neighbour (q = lower) or its lower neighbour (q = upper)
        if ((rc = write_val(s, p->pflags[q] + (q == 0 ? 2 : 1), sig))) return rc;
    }
    for (int q = 0; q < 2; ++q)
        if (has[q] && (rc = wait_geq(s, p->flags + 1 + q, sig, p->wait_flags))) return rc;
    return ST_OK;
}

static void clear_peer(stencil_s* h) {
    h->peer_lo = h->peer_hi = nullptr;
    h->peer_lo_end = h->peer_hi_begin = h->peer_d_lo = h->peer_d_hi = 0;
}

// One launch over all owned output planes: the halos are already in place
// (the stream waited for them), and the kernel itself stores the boundary
// planes into the neighbours, so there is nothing to overlap by splitting.
static int launch_owned(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s) {
    int64_t a, x0, x1, b;
    dist_output_slabs(h, &a, &x0, &x1, &b);
    return b > a ? launch_sweep(h, in, out, s, a, b) : ST_OK;
}

// stencil_step on a P2P-attached handle: exchange the input halos by peer
// copies (buffers must be registered), then compute.
int p2p_step(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s) {
    DistState* d = h->dist;
    P2PState* p = d->p2p;
    const unsigned mask = dist_halo_inputs(h->k->kind);
    int rc;
    // epochs: base = epoch+1 is skipped so that no stale "ready" signal of the
    // previous run (which equals epoch+1) can satisfy this exchange
    const uint32_t done_prev = p->epoch, sig = p->epoch + 2;
    for (int ai = 0; ai < h->k->n_in; ++ai) {
        if (!(mask >> ai & 1u)) continue;
        int k = -1;
        const PeerSet* ps = find_set(p, in[ai], &k);
        if (!ps) return set_error(ST_ESTATE, "input %d not registered with stencil_p2p_import", ai);
        if ((rc = exchange_inputs(h, ps, k, s, done_prev, sig))) return rc;
    }
    if ((rc = launch_owned(h, in, out, s))) return rc;
    p->epoch = sig;
    return write_val(s, p->flags, p->epoch);
}

int p2p_run(stencil_s* h, void* const* bufs, int n_iters, cudaStream_t s, int* result) {
    DistState* d = h->dist;
    P2PState* p = d->p2p;
    const KindInfo* k = h->k;
    int kidx = -1;
    const PeerSet* ps = find_set(p, bufs[0], &kidx);
    const int nb = k->iterable == 1 ? 2 : k->iterable == 2 ? 3 : k->n_in + k->n_out;
    if (!ps || kidx != 0 || ps->nb < nb) return set_error(ST_ESTATE, "run buffers not registered (stencil_p2p_import)");
    for (int a = 0; a < nb; ++a)
        if (ps->local[a] != bufs[a]) return set_error(ST_ESTATE, "run buffers differ from the registered set");
    const bool has[2] = {h->rank > 0, h->rank < h->nranks - 1};
    const int64_t m = d->m;
    const int lo = k->lo, hi = k->hi;
    const int64_t plane_elems = (int64_t)(d->plane_bytes / (h->dtype == ST_F64 ? 8 : 4));
    int rc;

    // prologue epochs: previous run ended at p->epoch (and signalled ready =
    // p->epoch+1 into buffers of that run); this run exchanges its current
    // field's halos with signal base+1, base = p->epoch+1, and its steps are
    // epochs base+1 ...
    const uint32_t done_prev = p->epoch, base = p->epoch + 1;
    if (!k->iterable) {                // static inputs: one exchange, then plain steps
        const unsigned mask = dist_halo_inputs(k->kind);
        for (int a = 0; a < k->n_in; ++a)
            if ((mask >> a & 1u) && (rc = exchange_inputs(h, ps, a, s, done_prev, base + 1))) return rc;
        const void* in[4];
        void* out[3];
        for (int a = 0; a < k->n_in; ++a) in[a] = bufs[a];
        for (int b = 0; b < k->n_out; ++b) out[b] = bufs[k->n_in + b];
        for (int it = 0; it < n_iters; ++it)
            if ((rc = launch_owned(h, in, out, s))) return rc;
        p->epoch = base + 1;
        if ((rc = write_val(s, p->flags, p->epoch))) return rc;
        *result = k->n_in;
        return ST_OK;
    }

    int idx[3] = {0, 1, 2};            // ping-pong (cur, next) or wave (prev, cur, next)
    const int cur0 = k->iterable == 1 ? 0 : 1;
    // prologue: the current field's halo planes from the neighbours first
    // (exchange_inputs returns once mine have arrived), then the Dirichlet
    // ring into the other run buffer(s).  In those buffers the fused peer
    // stores write only the interior columns of the halo planes, so the
    // x-edge (and, in 3-D, y-edge) cells of the halo planes come from this
    // ring copy, i.e. from the neighbours' values: the corner taps of the box
    // stencils read them.  Copying before the exchange arrived would
    // propagate whatever the caller left in the current field's halo planes.
    if ((rc = exchange_inputs(h, ps, cur0, s, done_prev, base + 1))) return rc;
    if (k->iterable == 1) {
        if ((rc = ring_copy(h, bufs[0], bufs[1], s))) return rc;
    } else {
        if ((rc = ring_copy(h, bufs[1], bufs[0], s))) return rc;
        if ((rc = ring_copy(h, bufs[1], bufs[2], s))) return rc;
    }
    p->epoch = base;
    if ((rc = write_val(s, p->flags, base))) return rc;
    for (int it = 0; it < n_iters; ++it) {
        const uint32_t e = p->epoch + 1;
        const int ic = k->iterable == 1 ? idx[0] : idx[1];
        const int io = k->iterable == 1 ? idx[1] : idx[2];
        for (int q = 0; q < 2; ++q)
            if (has[q]) {
                if ((rc = wait_geq(s, p->flags + 1 + q, e, p->wait_flags))) return rc;   // my input halos
                if ((rc = wait_geq(s, p->pflags[q], e - 1))) return rc;    // q's output buffer free
            }
        // fused stores of the output's boundary planes into the neighbours
        h->peer_lo = has[0] ? ps->peer[0][io] : nullptr;
        h->peer_hi = has[1] ? ps->peer[1][io] : nullptr;
        h->peer_lo_end = lo + hi;                      // my planes [lo, lo+hi) -> lower's [lo+m, ..)
        h->peer_d_lo = m * plane_elems;
        h->peer_hi_begin = m;                          // my planes [m, m+lo) -> upper's [0, lo)
        h->peer_d_hi = -m * plane_elems;
        const void* in[2];
        void* out[1] = {bufs[io]};
        if (k->iterable == 1) in[0] = bufs[ic];
        else { in[0] = bufs[idx[0]]; in[1] = bufs[ic]; }
        rc = launch_owned(h, in, out, s);
        clear_peer(h);
        if (rc) return rc;
        for (int q = 0; q < 2; ++q)
            if (has[q] && (rc = write_val(s, p->pflags[q] + (q == 0 ? 2 : 1), e + 1))) return rc;
        if ((rc = write_val(s, p->flags, e))) return rc;
        p->epoch = e;
        if (k->iterable == 1) std::swap(idx[0], idx[1]);
        else { const int t = idx[0]; idx[0] = idx[1]; idx[1] = idx[2]; idx[2] = t; }
    }
    *result = k->iterable == 1 ? idx[0] : idx[1];
    return ST_OK;
}

}  // namespace stb200

using namespace stb200;

namespace {
struct BlobRec {
    cudaIpcMemHandle_t handle;
    uint64_t offset;
};
constexpr uint32_t kBlobMagic = 0x53503250u;   // "P2PS"
}

extern "C" int stencil_dist_attach_p2p(stencil_t h, int rank, int nranks) {
    if (h && h->variant >= ST_PAPER_ORIGINAL)
        return set_error(ST_EUNSUPPORTED, "paper-literal variants cannot use the fused peer-store transport");
    if (!h) return set_error(ST_EARG, "null handle");
    if (!drv().ok) return set_error(ST_EUNSUPPORTED, "driver stream memory operations unavailable");
    int uva = 0, flush = 0;
    cudaDeviceGetAttribute(&uva, cudaDevAttrUnifiedAddressing, h->device);
    cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, h->device);
    if (!uva) return set_error(ST_EUNSUPPORTED, "device %d has no unified addressing (CUDA IPC peer pointers)",
                               h->device);
    DistState* d = nullptr;
    int rc = dist_attach_common(h, rank, nranks, &d);
    if (rc) return rc;
    d->p2p = new P2PState();
    if (flush) d->p2p->wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
    cudaError_t e = cudaMalloc(&d->p2p->flags, 256);
    if (e == cudaSuccess) e = cudaMemset(d->p2p->flags, 0, 256);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        h->dist = d;
        dist_release(h);
        return set_error(ST_ECUDA, "p2p flags: %s", cudaGetErrorString(e));
    }
    dist_attach_finish(h, d, rank, nranks);
    return ST_OK;
}

static int export_ptr(const void* ptr, BlobRec* r) {
    CUdeviceptr base = 0;
    size_t size = 0;
    if (drv().range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
        return set_error(ST_EARG, "cuMemGetAddressRange failed for %p", ptr);
    cudaError_t e = cudaIpcGetMemHandle(&r->handle, (void*)base);
    if (e != cudaSuccess) return set_error(ST_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    r->offset = (uint64_t)((const char*)ptr - (const char*)base);
    return ST_OK;
}

extern "C" int stencil_p2p_export(stencil_t h, void* const* bufs, int nbufs, uint8_t* blob, size_t cap,
                                  size_t* len) {
    if (!h || !h->dist || !h->dist->p2p) return set_error(ST_ESTATE, "handle not attached with stencil_dist_attach_p2p");
    if (!bufs || nbufs < 1 || nbufs > 8 || !blob || !len) return set_error(ST_EARG, "bad arguments");
    const size_t need = 8 + sizeof(BlobRec) * (size_t)(nbufs + 1);
    *len = need;
    if (cap < need) return set_error(ST_EARG, "blob capacity %zu < %zu", cap, need);
    uint32_t hdr[2] = {kBlobMagic, (uint32_t)nbufs};
    memcpy(blob, hdr, 8);
    BlobRec* rec = reinterpret_cast<BlobRec*>(blob + 8);
    int rc = export_ptr(h->dist->p2p->flags, &rec[0]);
    for (int k = 0; !rc && k < nbufs; ++k) rc = export_ptr(bufs[k], &rec[k + 1]);
    return rc;
}

static int open_rec(P2PState* p, const BlobRec& r, char** out) {
    const std::string key(reinterpret_cast<const char*>(&r.handle), sizeof r.handle);
    auto it = p->opened.find(key);
    if (it == p->opened.end()) {
        void* base = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&base, r.handle, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();        // not sticky; clear it for the caller's fallback
            return set_error(ST_EUNSUPPORTED, "cudaIpcOpenMemHandle: %s (no P2P path to the neighbour?)",
                             cudaGetErrorString(e));
        }
        // the mapping lives on the neighbour's device: it must be reachable
        // with peer loads / stores from this one (NVLink / NVSwitch)
        cudaPointerAttributes pa;
        int cur = -1, can = 1;
        cudaGetDevice(&cur);
        if (cudaPointerGetAttributes(&pa, base) == cudaSuccess && pa.device != cur && pa.device >= 0)
            cudaDeviceCanAccessPeer(&can, cur, pa.device);
        if (!can) {
            cudaIpcCloseMemHandle(base);
            return set_error(ST_EUNSUPPORTED, "device %d cannot access peer device %d", cur, pa.device);
        }
        it = p->opened.emplace(key, (char*)base).first;
    }
    *out = it->second + r.offset;
    return ST_OK;
}

extern "C" int stencil_p2p_import(stencil_t h, void* const* bufs, int nbufs, const uint8_t* lower,
                                  const uint8_t* upper) {
    if (!h || !h->dist || !h->dist->p2p) return set_error(ST_ESTATE, "handle not attached with stencil_dist_attach_p2p");
    if (!bufs || nbufs < 1 || nbufs > 8) return set_error(ST_EARG, "bad arguments");
    P2PState* p = h->dist->p2p;
    const uint8_t* blobs[2] = {h->rank > 0 ? lower : nullptr, h->rank < h->nranks - 1 ? upper : nullptr};
    PeerSet ps;
    ps.nb = nbufs;
    for (int k = 0; k < nbufs; ++k) ps.local[k] = bufs[k];
    cudaSetDevice(h->device);
    for (int q = 0; q < 2; ++q) {
        if (!blobs[q]) {
            if ((q == 0 && h->rank > 0) || (q == 1 && h->rank < h->nranks - 1))
                return set_error(ST_EARG, "missing neighbour blob");
            continue;
        }
        uint32_t hdr[2];
        memcpy(hdr, blobs[q], 8);
        if (hdr[0] != kBlobMagic || (int)hdr[1] != nbufs) return set_error(ST_EARG, "neighbour blob mismatch");
        const BlobRec* rec = reinterpret_cast<const BlobRec*>(blobs[q] + 8);
        char* f = nullptr;
        int rc = open_rec(p, rec[0], &f);
        if (rc) return rc;
        p->pflags[q] = reinterpret_cast<uint32_t*>(f);
        for (int k = 0; k < nbufs; ++k)
            if ((rc = open_rec(p, rec[k + 1], &ps.peer[q][k]))) return rc;
    }
    // replace an older registration of the same first buffer
    for (auto it = p->sets.begin(); it != p->sets.end(); ++it)
        if (it->local[0] == bufs[0]) { p->sets.erase(it); break; }
    p->sets.push_back(ps);
    return ST_OK;
}
