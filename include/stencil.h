/*
 * stencil.h — C ABI of the B200-native register-cache stencil library
 * (libstencil_b200.so).  No C++, CUDA-runtime or torch types cross this
 * boundary: handles are opaque pointers, device buffers are plain `void*`
 * device pointers, CUDA streams are passed as `void*` (a cudaStream_t value;
 * NULL = the legacy default stream).
 *
 * What is computed (arxiv 2301.11389): the stencil / neighbour-access loop
 * nests of the KernelGen OpenACC suite (Table 1) whose
 * overlapping neighbour loads PTXASW replaces by warp shuffles
 * (§5.1 "Detection", 503-518; §5.2 "Code Generation", 523-576).
 * The only formula the paper prints is the 9-point Jacobi of Listing 5
 * (PAPER.md:405-415); the readings of the other kinds are in DESIGN.md §3.
 * Every kernel evaluates the out-of-place, interior-only loop nest of
 * Listing 5 ("updates different arrays").
 *
 * Layout: dense, contiguous, x fastest (x = the thread dimension, "leading
 * dimension").  2-D element (i,j) at j*nx+i; 3-D (i,j,k)
 * at (k*ny+j)*nx+i.  `dims` = {nx, ny[, nz]} include the boundary ring.
 * One dtype per handle.  Every buffer must be 16-byte aligned and
 * nx*sizeof(T) % 16 == 0 (whole 16-byte vectors per row), else ST_EALIGN.
 *
 * Ownership: the caller owns every device and host buffer; the library never
 * allocates or frees them.  A handle owns its configuration, coefficients,
 * cached CUDA graphs, an internal capture stream and (after
 * stencil_dist_attach) an NCCL communicator — all released by
 * stencil_destroy.  A handle is not thread-safe; distinct handles are
 * independent.
 *
 * Errors: every call returns ST_OK (0) or a negative status; a detail string
 * is available from stencil_last_error() (thread-local, valid until the next
 * failing call on the same thread).  Calls only enqueue device work on the
 * given stream: launch errors are returned immediately (ST_ECUDA);
 * asynchronous device faults surface as sticky CUDA errors on a later call.
 */
#ifndef STENCIL_B200_H
#define STENCIL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stencil_s* stencil_t;

/* Kinds.  Arity (inputs -> outputs) and halo radius lo/hi per axis:
 *  ST_JACOBI2D5     in -> out, r=1   Listing 5 without the c2 term      coeffs (c0,c1)       default (0, 1/4)
 *  ST_JACOBI2D9     in -> out, r=1   Listing 5       coeffs (c0,c1,c2)    default (1/4,1/8,1/16)
 *  ST_GAUSSBLUR5X5  in -> out, r=2   Table 1 gaussblur, 25 loads        25 weights w[dj][di] default binomial/256
 *                   (rank-1 weights are factored at create, w = u v^T: the
 *                   register-cache kernels then run a 5-tap row pass and a
 *                   5-tap column pass, equal to the 25-term sum up to rounding)
 *  ST_GAMEOFLIFE    in -> out, r=1   Table 1 gameoflife, int32 B3/S23   none
 *                   (cells are Life states 0 / 1; the streaming multi-sweep
 *                   kernel packs four cells per register and reads a cell as
 *                   its lowest bit, so only 0/1 grids are defined)
 *  ST_LAPLACIAN3D7  in -> out, r=1   Table 1 laplacian, 7 loads         coeffs (a,b)         default (-6, 1)
 *  ST_JACOBI3D7     in -> out, r=1   laplacian form, Jacobi weights     coeffs (a,b)         default (0, 1/6)
 *  ST_WAVE13PT      (prev,cur) -> next, r=2  Table 1 wave13pt, 14 loads coeffs (m0,m1,m2)    default lambda=1/8
 *  ST_DIVERGENCE    (u,v,w) -> out, r=1      Table 1 divergence         coeffs (ax,ay,az)    default (1/2,1/2,1/2)
 *  ST_GRADIENT      u -> (gx,gy,gz), r=1     Table 1 gradient           coeffs (ax,ay,az)    default (1/2,1/2,1/2)
 *  ST_TRICUBIC      (f,X,Y,Z) -> g, lo=1 hi=2  Table 1 tricubic, 67 loads none
 * SURVEY §8(f) row f3 (readings DESIGN.md §3 R19-R22; PAPER.md prints no formula):
 *  ST_TRICUBIC2     (f,X,Y,Z) -> g, lo=1 hi=2  Table 1 tricubic2: tricubic as the
 *                   expanded 64-term sum; the same function up to rounding   none
 *  ST_UXX1          (u1,d1,xx,xy,xz) -> u1', lo=2 hi=1  Table 1 uxx1: 4th-order
 *                   staggered velocity update, 17 loads             coeffs (dth,c1,c2)   default (1/4, 9/8, -1/24)
 *  ST_LAPGSRB       u -> u', r=1  Table 1 lapgsrb: one red-black Gauss-Seidel
 *                   iteration of the 7-point Laplace operator, 25 loads (L1 ball of radius 2)
 *                                                                   coeffs (w)           default 1/6
 *  ST_WHISPERING    (Hx,Hy,Ez,dax,dbx,day,dby,cb) -> (Hx',Hy',Ez'), 2-D, r=1  Table 1 whispering
 *                   (PAPER.md:608): one fused TM-mode Yee (FDTD) leapfrog step, 19 loads   none
 * The f3 kinds run on one GPU (stencil_dist_attach*: ST_EUNSUPPORTED) with the
 * SHUFFLE / PLAIN variants (paper-literal variants: ST_EUNSUPPORTED).
 * Formulas: DESIGN.md §3 (and oracle/oracle.c, the independent CPU oracle). */
enum stencil_kind {
    ST_JACOBI2D5 = 1, ST_JACOBI2D9 = 2, ST_GAUSSBLUR5X5 = 3, ST_GAMEOFLIFE = 4,
    ST_LAPLACIAN3D7 = 5, ST_JACOBI3D7 = 6, ST_WAVE13PT = 7, ST_DIVERGENCE = 8,
    ST_GRADIENT = 9, ST_TRICUBIC = 10,
    ST_TRICUBIC2 = 11, ST_UXX1 = 12, ST_LAPGSRB = 13, ST_WHISPERING = 14
};

/* Element types.  ST_I32 only for ST_GAMEOFLIFE; the others take F32/F64. */
enum stencil_dtype { ST_F32 = 1, ST_F64 = 2, ST_I32 = 3 };

/* Kernel variants, the paper's question "does the shuffle pay?" (PAPER.md
 * §7-8) asked on Blackwell.  Both variants are register-blocked (each lane
 * owns one 16-byte vector of a warp row tile) and give bit-identical results.
 *  ST_SHUFFLE: x-neighbour taps outside a lane's vector come from lanes l-1 /
 *              l+1 by shfl.sync.up/down; warp-edge lanes
 *              fall back to a predicated load (the %out_of_range corner case,
 *              PAPER.md:561-564).
 *  ST_PLAIN:   the same taps come from loads (L1 / shared memory), i.e. the
 *              original code's loads, no shuffles.
 * The paper-literal family (every kind in fp32/int32 only: the paper
 * shuffles 32-bit data; not with the fused peer-store
 * transport, ST_EUNSUPPORTED): one output per thread, 512 threads per
 * block along x (Listing 5), leftmost tap of each x-row as
 * the shuffle source, written as the PTX of Listing 6:
 *  ST_PAPER_ORIGINAL: every tap an ld.global.nc (the compiler's code)
 *  ST_PAPER_PTXASW:   activemask / %incomplete / %out_of_range / or.pred,
 *                     shfl.sync.down at the load site, @pred original load
 *  ST_PAPER_NOLOAD:   covered loads removed (INVALID results)
 *  ST_PAPER_NOCORNER: shuffles without corner fallback (INVALID at warp edges)
 *  ST_PAPER_UNIFORM:  warp-uniform branch on completeness
 * Bit-identical to SHUFFLE/PLAIN except NOLOAD and NOCORNER.
 *  ST_AUTO: resolved by stencil_set_variant, per kind, to whichever of
 *           SHUFFLE / PLAIN ran faster on B200 at the kind's benchmark size
 *           (the answer differs by kind); stencil_get_variant
 *           then reports the resolved variant. */
enum stencil_variant {
    ST_SHUFFLE = 0, ST_PLAIN = 1,
    ST_PAPER_ORIGINAL = 2, ST_PAPER_PTXASW = 3, ST_PAPER_NOLOAD = 4, ST_PAPER_NOCORNER = 5,
    ST_PAPER_UNIFORM = 6, ST_AUTO = 7
};

enum stencil_status {
    ST_OK = 0,
    ST_EARG = -1,          /* bad argument (null, size, aliasing, count)          */
    ST_EUNSUPPORTED = -2,  /* kind/dtype/variant combination not provided         */
    ST_EALIGN = -3,        /* pointer not 16-B aligned or nx*sizeof(T) % 16 != 0   */
    ST_ECUDA = -4,         /* CUDA runtime/launch error (detail in last_error)    */
    ST_ENCCL = -5,         /* NCCL error or NCCL library not loadable             */
    ST_ESTATE = -6         /* call not valid in the handle's current state        */
};

/* Create a handle.  dims[ndims] = {nx, ny[, nz]} (global dims if the handle
 * is later attached to a multi-GPU group).  Each axis must be >= lo+hi+1
 * (at least one interior point).  coeffs: ncoeffs == 0 selects the defaults
 * above, otherwise ncoeffs must equal the kind's count; values are converted
 * to the handle's dtype.  Returns ST_EARG / ST_EUNSUPPORTED / ST_EALIGN. */
int stencil_create(stencil_t* h, int kind, int ndims, const int64_t* dims, int dtype,
                   const double* coeffs, int ncoeffs);

/* Select the kernel variant for subsequent calls (default ST_SHUFFLE);
 * ST_EUNSUPPORTED for a paper-literal variant on a 3-D or fp64 handle. */
int stencil_set_variant(stencil_t h, int variant);
int stencil_get_variant(stencil_t h, int* variant);

/* Temporal blocking of 2-D ping-pong runs: stencil_run may
 * apply several sweeps per kernel launch; results are bit-identical to
 * single sweeps.
 *   0 (default) auto: grids that sit in L2 (<= 8 MiB per buffer) run the
 *                     on-chip kernels (per-launch latency bounds those runs);
 *                     larger jacobi2d5 / gameoflife grids run the streaming
 *                     three-sweep register-cache kernel, jacobi2d9 and
 *                     gaussblur with separable (rank-1) weights — the default
 *                     binomial — the two-sweep one (one HBM pass per two or
 *                     three sweeps: the single-sweep kernel is HBM-bound); a
 *                     gaussblur with non-separable weights keeps one sweep per
 *                     launch (issue-bound at two sweeps per pass: no gain)
 *   1           never fuse (one sweep per launch)
 *   2           the streaming kernel with exactly two sweeps per launch
 *   3           the streaming kernel with exactly three sweeps per launch
 *               (jacobi2d5 / jacobi2d9 / gameoflife / separable gaussblur5x5;
 *               ST_EUNSUPPORTED for gaussblur5x5 with non-separable weights)
 *   -S (S >= 2) the shared-memory tile kernel, at most S sweeps per launch
 * A run whose sweep count is not a multiple of the streaming depth runs the
 * remainder as single sweeps first.  Anything else: ST_EARG.  Only the
 * register-cache variants (SHUFFLE/PLAIN) and single-GPU handles fuse;
 * stencil_step is always one sweep.  The result buffer of a run is reported
 * in *result_idx (fused runs may differ from n_iters % 2); the other buffer
 * holds an earlier sweep. */
int stencil_set_fusion(stencil_t h, int sweeps_per_launch);

/* Arity: inputs and outputs of one step; buffers stencil_run expects
 * (2 for ping-pong kinds, 3 for wave13pt, n_in+n_out for the others). */
int stencil_arity(stencil_t h, int* n_in, int* n_out, int* n_bufs_for_run);

/* Static description of the handle, for benchmarks and tests. */
typedef struct {
    int kind, dtype, ndims, variant;
    int64_t dims[3];          /* global dims                                        */
    int64_t local_dims[3];    /* this rank's buffer dims (== dims when not attached) */
    int lo, hi;               /* halo radius below / above, every axis              */
    int64_t interior_points;  /* points one step writes on this rank                */
    double bytes_per_point;   /* compulsory HBM bytes per interior point per step   */
    int launches_per_step;    /* kernels one stencil_step enqueues                  */
    int sweeps_per_launch;    /* sweeps per sweep-kernel launch of a long stencil_run
                                 on this handle (1, 2 / 3 = streaming, S = tile)   */
    int rank, nranks;         /* 0,1 unless attached                                */
} stencil_info_t;
int stencil_info(stencil_t h, stencil_info_t* out);

/* One application: out[a] <- kind(in[0..n_in)) at interior points only; the
 * boundary ring of out is never written.  in/out arrays hold n_in / n_out
 * device pointers of `local_dims` elements; no out may alias an in
 * (ST_EARG).  Multi-GPU (attached): exchanges the halo planes of in[] with
 * the neighbour ranks (NCCL send/recv, overlapped with the interior); the
 * halo planes of the inputs are overwritten by the exchange. */
int stencil_step(stencil_t h, const void* const* in, void* const* out, void* stream);

/* Like stencil_step on one GPU, but writes only the output planes
 * [s_begin, s_end) of the slow axis (z in 3-D, y in 2-D) of the local
 * buffers; lo <= s_begin <= s_end <= local_n - hi, else ST_EARG.  No halo
 * exchange.  The building block of the overlapped multi-GPU step (interior
 * slab while the halo is in flight, then the halo-dependent slabs) and of
 * user-level decompositions. */
int stencil_step_range(stencil_t h, const void* const* in, void* const* out,
                       int64_t s_begin, int64_t s_end, void* stream);

/* n_iters sweeps ("running the ... kernel ten times"): copies the
 * current field's boundary ring into the other buffers once (Dirichlet), then
 * enqueues the sweeps as one cached CUDA graph on `stream`.
 *   ping-pong kinds: bufs = {A, B}, current = A; result in bufs[*result_idx].
 *   wave13pt:        bufs = {prev, cur, next}; rotation (prev,cur,next) <-
 *                    (cur,next,prev) after each sweep; result = current level.
 *   others:          bufs = {inputs..., outputs...}; the same step repeated.
 * Graphs are cached per (bufs, n_iters, variant); n_iters == 0 only copies. */
int stencil_run(stencil_t h, void* const* bufs, int n_iters, void* stream, int* result_idx);

/* End-to-end form of stencil_run with HOST buffers: copies host_in[0..n_in)
 * (pinned or pageable host memory, local_dims elements each) into dev_bufs,
 * runs n_iters sweeps, copies the result buffer(s) back to host_out[0..n_out)
 * and synchronises `stream`.  dev_bufs is the caller-owned device workspace
 * with the layout stencil_run expects (for wave13pt host_in = {prev, cur}). */
int stencil_run_host(stencil_t h, const void* const* host_in, void* const* host_out,
                     void* const* dev_bufs, int n_iters, void* stream);

/* stencil_run_host without the final synchronisation: the H2D copies, the
 * run and the D2H copies are only enqueued on `stream` (completion is the
 * caller's stream sync or event).  Host buffers must be pinned for the
 * copies to be asynchronous, and must stay valid until the stream reaches
 * them.  With two handles, two device workspaces and two streams, the
 * copies of one run overlap the sweeps of the other (bench.py e2e). */
int stencil_run_host_async(stencil_t h, const void* const* host_in, void* const* host_out,
                           void* const* dev_bufs, int n_iters, void* stream);

int stencil_destroy(stencil_t h);

/* Thread-local description of the last failure on this thread. */
const char* stencil_last_error(void);

/* Library version string and the SASS architecture it was built for. */
const char* stencil_version(void);

/* ---------------------------------------------------------------- multi-GPU
 * 1-D slab decomposition along the slowest axis (z in 3-D, y in 2-D), one
 * process per GPU.  Rank p owns global planes [p*n/N, (p+1)*n/N) of the
 * interior-inclusive axis (n = the slow dim, divisible by N) and holds
 * lo + n/N + hi planes locally; the outermost ranks' extra planes are the
 * global Dirichlet boundary.  Results are bit-identical to one GPU. */

/* Host-only plan (no GPU needed): for global slow extent n, halo lo/hi,
 * rank/nranks, fills plan[8] = {own_begin, own_end, local_n, recv_lo_at,
 * send_lo_from, recv_hi_at, send_hi_from, n_planes_lo | n_planes_hi << 16}
 * in local plane indices (-1 where there is no neighbour).  ST_EARG if n is
 * not divisible by nranks or a slab is thinner than the halo. */
int stencil_slab_plan(int64_t n, int lo, int hi, int rank, int nranks, int64_t plan[8]);

/* NCCL unique id for the group (call on rank 0, broadcast the 128 bytes with
 * torch.distributed, then attach on every rank).  ST_ENCCL if libnccl.so.2
 * cannot be loaded. */
int stencil_dist_get_id(uint8_t id[128]);

/* Join the group: creates the NCCL communicator for this handle on the
 * current device; afterwards local buffers have local_dims (see
 * stencil_info) and stencil_step/stencil_run exchange halos internally. */
int stencil_dist_attach(stencil_t h, const uint8_t id[128], int rank, int nranks);

/* Host transport for the halo exchange, instead of NCCL (tests, or
 * deployments that move the planes with MPI / another library): the library
 * copies the planes to pinned host memory and calls, for each neighbour,
 *   fn(peer, send, send_bytes, recv, recv_bytes, user)
 * which must send `send` to rank `peer` and receive `recv_bytes` from it
 * into `recv` (host pointers; return 0 on success).  Synchronous: no
 * overlap with the interior.  Same slab layout and results as
 * stencil_dist_attach. */
typedef int (*stencil_exchange_fn)(int peer, const void* send, size_t send_bytes, void* recv,
                                   size_t recv_bytes, void* user);
int stencil_dist_attach_host(stencil_t h, int rank, int nranks, stencil_exchange_fn fn, void* user);

/* Fused halo exchange over peer memory (the "compute + collective in one
 * kernel" transport): the kernels that compute a rank's boundary planes also
 * store them straight into the neighbours' buffers through CUDA-IPC peer
 * pointers (NVLink / NVSwitch P2P), and ranks order themselves with epoch
 * flags in device memory (stream memory operations, no spinning SMs).
 *   1. stencil_dist_attach_p2p(h, rank, nranks)
 *   2. for a set of run buffers: stencil_p2p_export writes a blob (IPC
 *      handles of the rank's flags and buffers); all-gather the blobs (e.g.
 *      torch.distributed); stencil_p2p_import(h, bufs, n, blob of rank-1,
 *      blob of rank+1) maps the neighbours' buffers (NULL where none)
 *   3. stencil_run / stencil_step with exactly those buffers.
 * Buffers must be plain device allocations (cudaMalloc / torch default
 * allocator).  Same slab layout and results as stencil_dist_attach. */
int stencil_dist_attach_p2p(stencil_t h, int rank, int nranks);
int stencil_p2p_export(stencil_t h, void* const* bufs, int nbufs, uint8_t* blob, size_t cap, size_t* len);
int stencil_p2p_import(stencil_t h, void* const* bufs, int nbufs, const uint8_t* lower_blob,
                       const uint8_t* upper_blob);

#ifdef __cplusplus
}
#endif
#endif /* STENCIL_B200_H */
