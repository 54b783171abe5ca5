// pipe.cuh — Blackwell async-copy primitives: mbarrier + cp.async.bulk
// (the bulk-copy path of the Tensor Memory Accelerator, SASS UBLKCP) and the
// TMA tensor copy (cp.async.bulk.tensor, SASS UTMALDG).  Inline PTX only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace stb200 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// Make barrier initialisation visible to the async proxy (TMA unit).
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Order this thread's prior generic-proxy shared-memory accesses before
// subsequent async-proxy (bulk copy) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One arrival that also announces `bytes` of transaction (completed by TMA).
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Consumer release of a ring stage right after this thread's shared-memory
// loads from it were ISSUED.  Measured on B200: a plain
// arrive issued behind in-flight LDS lets the producer's next bulk copy
// overwrite the stage before those loads read it (PLAIN gaussblur 8192^2
// x100 differed run to run).  The release is ordered by a cross-proxy fence
// (fence.proxy.async: the thread's generic-proxy reads of the stage before
// the async-proxy writes the producer issues after this arrival).
// STB200_REL (build knob): 1 = fence.proxy.async + arrive (default); 2 =
// the round-1 data-dependency form (`dep`, 0 at run time but computed from
// the loaded registers, added to the barrier address) — it was NOT enough:
// jacobi2d5 32768^2 three-sweep PLAIN and jacobi2d9 two-sweep runs still
// differed run to run (tools/flake_hunt.py, round 2), the fenced form is
// clean; 0 = plain arrive (racy, A/B only).
#ifndef STB200_REL
#define STB200_REL 1
#endif
// Streaming row rings (k2d, k2d2, klife): the stage of row r is released at
// the START of consume(r + 1), fenced — by then row r's loads have been
// consumed by the arithmetic, so the proxy fence has nothing left to wait
// for (releasing right after the loads, fenced, cost 6-10% on the PLAIN
// variants).  0 = release right after the loads (STB200_REL form).
#ifndef STB200_REL_LAG
#define STB200_REL_LAG 1
#endif
// ... in batches of B rows per fence (consume(r), r % B == 0, releases rows
// r-B .. r-1 behind one fence).  Measured (round 2, tools/gpu_lag_ab.sh):
// B = 4 helps the PLAIN kernels (gaussblur 1165 -> 1213, jacobi2d5 three-sweep
// 1531 -> 1627 Gpt/s), B = 1 suits SHUFFLE (1214 / 1911 vs 1206 / 1846):
// the kernels pass B per variant.  STB200_REL_BATCH overrides (A/B builds).
#ifndef STB200_REL_BATCH
#define STB200_REL_BATCH 0
#endif
// D > 0 keeps D more rows resident (released D rows later): k2d2 re-reads
// the raw input row of a window centre for the held boundary-ring values.
template <unsigned S, unsigned B0 = 1, unsigned D = 0>
__device__ __forceinline__ void ring_release_lagged(uint64_t* empty, unsigned r_) {
    constexpr unsigned B = STB200_REL_BATCH > 0 ? STB200_REL_BATCH : B0;
    static_assert(D + B < S, "the producer needs a free stage");
    if (r_ < D) return;
    const unsigned r = r_ - D;
    if (r == 0 || r % B != 0) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (unsigned q = r - B; q < r; ++q)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[q & (S - 1)])) : "memory");
}
__device__ __forceinline__ void mbar_release(uint64_t* bar, uint32_t dep) {
    uint32_t a = smem_u32(bar);
    if (STB200_REL == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (STB200_REL == 2) a += dep;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// The same release ordered by a proxy fence instead of a data dependency:
// the thread's earlier generic-proxy shared-memory reads are ordered before
// the async-proxy writes the producer issues after this arrival.
__device__ __forceinline__ void mbar_release_fenced(uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t bits32(float x) { return __float_as_uint(x); }
__device__ __forceinline__ uint32_t bits32(int x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t bits32(double x) { return (uint32_t)__double_as_longlong(x); }

// Block until the barrier's phase with the given parity has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Wait used by producer warps: back off between polls (exponentially, up
// to MAXNS ns) so that a producer waiting for the consumers to free a stage
// does not take issue slots from the consumer warps of its SM sub-partition.
template <uint32_t MAXNS>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    uint32_t ok, ns = 32;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (ok) return;
        __nanosleep(ns);
        if (ns < MAXNS) ns *= 2;
    }
}

// Bulk copy global -> shared (contiguous, 16-byte aligned, bytes % 16 == 0),
// completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Bulk copy shared -> global (contiguous, 16-byte aligned, bytes % 16 ==
// 0) in the issuing thread's bulk group; the source may be reused once
// bulk_wait_read has returned in the same thread.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Thread t's earlier bulk stores have finished reading shared memory; then
// the warp may overwrite the staging rows.
__device__ __forceinline__ void bulk_wait_read(bool t) {
    if (t) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
}
__device__ __forceinline__ void bulk_wait_all(bool t) {
    if (t) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
}

// L2 eviction-first policy for streamed data read exactly once.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
        "%2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// TMA tensor load of a 3-D box (coordinates x fastest; out-of-bounds parts
// of the box are zero-filled) into shared memory, completion on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

}  // namespace stb200
