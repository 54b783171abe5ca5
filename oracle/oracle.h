/*
 * oracle.h — plain, slow, obviously-correct CPU oracle for the stencil loop
 * nests whose redundant neighbour loads PTXASW replaces by warp shuffles
 * (arxiv 2301.11389, §6 "Experimental Methodology", Table 1,
 * PAPER.md:593-617; the only printed formula is Listing 5).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2301_11389_b200/csrc, include/stencil.h) and includes nothing
 * from it.  Kinds and dtypes are passed as strings so that not even an
 * enum is shared.
 *
 * Every floating-point result is computed in double (fp64) from the
 * stored inputs and rounded once to the grid's storage type when stored
 * ("f32" grids store float, "f64" grids double).  "i32" (gameoflife) is
 * integer arithmetic.  Compiled with -O2 -ffp-contract=off (no FMA
 * contraction, no reassociation): each formula is evaluated left to right
 * exactly as written in DESIGN.md §3.
 *
 * Layout: dense, x fastest.  2-D a[j][i] at j*nx+i; 3-D a[k][j][i] at
 * (k*ny+j)*nx+i.  dims = {nx, ny[, nz]} include the boundary ring.
 * A step writes interior points only: lo <= i < nx-hi (same for j, k);
 * Listing 5 loop bounds j=2..ny-1, i=2..nx-1 (1-based Fortran),
 * PAPER.md:409-411.
 *
 * Return codes: 0 ok, -1 bad argument (message via oracle_error()).
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Shape of a kind: inputs, outputs, buffers for oracle_run, halo lo/hi. */
int oracle_arity(const char* kind, int* n_in, int* n_out, int* n_bufs,
                 int* lo, int* hi, int* ndims, int* ncoeffs);

/* Default coefficients of a kind (DESIGN.md §3 reading R2). */
int oracle_default_coeffs(const char* kind, double* out, int cap);

/* One application: out[] <- stencil(in[]) on interior points only. */
int oracle_step(const char* kind, const char* dtype, int ndims,
                const int64_t* dims, const double* coeffs, int ncoeffs,
                const void* const* in, void* const* out, int nthreads);

/* n_iters applications with Dirichlet boundary (ring copied once from the
 * current field into the other buffers first).  Iterable kinds ping-pong
 * bufs[0]<->bufs[1]; wave13pt rotates (prev,cur,next) <- (cur,next,prev);
 * divergence/gradient/tricubic re-apply the same step (benchmark mode,
 * "running the ... kernel ten times").  *result_idx = index
 * into bufs of the buffer holding the (first) result. */
int oracle_run(const char* kind, const char* dtype, int ndims,
               const int64_t* dims, const double* coeffs, int ncoeffs,
               void* const* bufs, int n_iters, int nthreads, int* result_idx);

const char* oracle_error(void);

#ifdef __cplusplus
}
#endif
#endif
