/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h for who may load it).
 *
 * The plain definition of every stencil of the hot path, evaluated
 * literally in fp64 (int for gameoflife), one point at a time, with no
 * blocking, fusion or reordering.  The method being accelerated (register
 * caching via warp shuffles, §5) only relocates loaded bits and
 * changes no arithmetic ("the shuffle operation is performed
 * at the position of the original load"), so the oracle is the plain loop
 * nest of each KernelGen benchmark (Table 1).
 *
 * Which passage each function follows is stated at the function.  Where
 * PAPER.md names a benchmark but does not print its formula, the reading
 * is DESIGN.md §3 (R1..R12) and is stated at the function too.
 */
#include "oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[256];
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
const char* oracle_error(void) { return g_err; }

/* ---------------------------------------------------------------- types */
enum { DT_F32, DT_F64, DT_I32, DT_BAD };
static int parse_dtype(const char* s) {
    if (!s) return DT_BAD;
    if (!strcmp(s, "f32")) return DT_F32;
    if (!strcmp(s, "f64")) return DT_F64;
    if (!strcmp(s, "i32")) return DT_I32;
    return DT_BAD;
}
static size_t dt_size(int dt) { return dt == DT_F64 ? 8 : 4; }

/* Read element idx of array p as double (exact for f32/f64/i32). */
static double rd(const void* p, int dt, int64_t idx) {
    if (dt == DT_F32) return (double)((const float*)p)[idx];
    if (dt == DT_F64) return ((const double*)p)[idx];
    return (double)((const int32_t*)p)[idx];
}
/* Store a double result, rounded once to the storage type. */
static void wr(void* p, int dt, int64_t idx, double v) {
    if (dt == DT_F32) ((float*)p)[idx] = (float)v;
    else if (dt == DT_F64) ((double*)p)[idx] = v;
    else ((int32_t*)p)[idx] = (int32_t)v;
}

/* ---------------------------------------------------------------- kinds */
typedef struct {
    const char* name;
    int ndims, n_in, n_out, lo, hi, ncoeffs, iterable; /* iterable: 1 ping-pong, 2 three-level */
    int allow_f, allow_i;
} kind_t;

static const kind_t KINDS[] = {
    /* name            nd in out lo hi nc it  f  i */
    {"jacobi2d5",       2, 1, 1, 1, 1, 2, 1, 1, 0},
    {"jacobi2d9",       2, 1, 1, 1, 1, 3, 1, 1, 0},
    {"gaussblur5x5",    2, 1, 1, 2, 2, 25, 1, 1, 0},
    {"gameoflife",      2, 1, 1, 1, 1, 0, 1, 0, 1},
    {"laplacian3d7",    3, 1, 1, 1, 1, 2, 1, 1, 0},
    {"jacobi3d7",       3, 1, 1, 1, 1, 2, 1, 1, 0},
    {"wave13pt",        3, 2, 1, 2, 2, 3, 2, 1, 0},
    {"divergence",      3, 3, 1, 1, 1, 3, 0, 1, 0},
    {"gradient",        3, 1, 3, 1, 1, 3, 0, 1, 0},
    {"tricubic",        3, 4, 1, 1, 2, 0, 0, 1, 0},
    /* SURVEY §8(f) row f3 (DESIGN.md §3 readings R19-R22) */
    {"tricubic2",       3, 4, 1, 1, 2, 0, 0, 1, 0},
    {"uxx1",            3, 5, 1, 2, 1, 3, 0, 1, 0},
    {"lapgsrb",         3, 1, 1, 1, 1, 1, 1, 1, 0},
    {"whispering",      2, 8, 3, 1, 1, 0, 0, 1, 0},
};

static const kind_t* find_kind(const char* name) {
    if (!name) return NULL;
    for (size_t i = 0; i < sizeof KINDS / sizeof KINDS[0]; ++i)
        if (!strcmp(KINDS[i].name, name)) return &KINDS[i];
    return NULL;
}

int oracle_arity(const char* kind, int* n_in, int* n_out, int* n_bufs,
                 int* lo, int* hi, int* ndims, int* ncoeffs) {
    const kind_t* k = find_kind(kind);
    if (!k) return fail("unknown kind");
    if (n_in) *n_in = k->n_in;
    if (n_out) *n_out = k->n_out;
    if (n_bufs) *n_bufs = k->iterable == 1 ? 2 : k->iterable == 2 ? 3 : k->n_in + k->n_out;
    if (lo) *lo = k->lo;
    if (hi) *hi = k->hi;
    if (ndims) *ndims = k->ndims;
    if (ncoeffs) *ncoeffs = k->ncoeffs;
    return 0;
}

/* Default coefficients, DESIGN.md §3 reading R2 (the paper prints only the
 * symbols c0,c1,c2 of Listing 5, never their values). */
int oracle_default_coeffs(const char* kind, double* out, int cap) {
    const kind_t* k = find_kind(kind);
    if (!k) return fail("unknown kind");
    if (cap < k->ncoeffs) return fail("capacity too small");
    const char* n = k->name;
    if (!strcmp(n, "jacobi2d5")) { out[0] = 0.0; out[1] = 0.25; }
    else if (!strcmp(n, "jacobi2d9")) { out[0] = 0.25; out[1] = 0.125; out[2] = 0.0625; }
    else if (!strcmp(n, "gaussblur5x5")) {
        /* binomial [1,4,6,4,1]^T [1,4,6,4,1] / 256 */
        const double b[5] = {1, 4, 6, 4, 1};
        for (int dj = 0; dj < 5; ++dj)
            for (int di = 0; di < 5; ++di) out[dj * 5 + di] = b[dj] * b[di] / 256.0;
    }
    else if (!strcmp(n, "laplacian3d7")) { out[0] = -6.0; out[1] = 1.0; }
    else if (!strcmp(n, "jacobi3d7")) { out[0] = 0.0; out[1] = 1.0 / 6.0; }
    else if (!strcmp(n, "wave13pt")) {
        /* leapfrog wave equation, 4th-order Laplacian, lambda = c^2 dt^2/h^2 = 1/8:
         * m0 = 2 - 7.5*lambda, m1 = 4*lambda/3, m2 = -lambda/12 */
        const double lam = 0.125;
        out[0] = 2.0 - 7.5 * lam; out[1] = 4.0 * lam / 3.0; out[2] = -lam / 12.0;
    }
    else if (!strcmp(n, "divergence") || !strcmp(n, "gradient")) { out[0] = out[1] = out[2] = 0.5; }
    else if (!strcmp(n, "uxx1")) {
        /* (dth, c1, c2): dth = dt/h (R20: a value of the reading), c1 = 9/8,
         * c2 = -1/24 the 4th-order staggered-grid difference weights */
        out[0] = 0.25; out[1] = 9.0 / 8.0; out[2] = -1.0 / 24.0;
    }
    else if (!strcmp(n, "lapgsrb")) { out[0] = 1.0 / 6.0; }   /* Gauss-Seidel weight of the 7-point Laplace operator */
    return k->ncoeffs;
}

/* ------------------------------------------------------------ geometry */
typedef struct {
    int64_t nx, ny, nz;
    int dt;
} geom_t;

static int64_t I2(const geom_t* g, int64_t j, int64_t i) { return j * g->nx + i; }
static int64_t I3(const geom_t* g, int64_t k, int64_t j, int64_t i) {
    return (k * g->ny + j) * g->nx + i;
}

/* ----------------------------------------------- 2-D point definitions */

/* jacobi2d9 — Listing 5, Fortran w1(i,j) with
 * w0(i+-1, j+-1) mapped to in[j][i] (x = i fastest):
 *   w1(i,j)=c0*w0(i,j) + c1*(w0(i-1,j)+w0(i,j-1)+w0(i+1,j)+w0(i,j+1))
 *         + c2*(w0(i-1,j-1)+w0(i-1,j+1)+w0(i+1,j-1)+w0(i+1,j+1))        */
static double pt_jacobi2d9(const geom_t* g, const void* in, const double* c,
                           int64_t j, int64_t i) {
    const int dt = g->dt;
    return c[0] * rd(in, dt, I2(g, j, i))
         + c[1] * (rd(in, dt, I2(g, j, i - 1)) + rd(in, dt, I2(g, j - 1, i))
                   + rd(in, dt, I2(g, j, i + 1)) + rd(in, dt, I2(g, j + 1, i)))
         + c[2] * (rd(in, dt, I2(g, j - 1, i - 1)) + rd(in, dt, I2(g, j + 1, i - 1))
                   + rd(in, dt, I2(g, j - 1, i + 1)) + rd(in, dt, I2(g, j + 1, i + 1)));
}

/* jacobi2d5 — Listing 5 with the c2 (diagonal) term removed: the 5-point
 * form named by BASELINE configs[0] (DESIGN.md §3 reading R3). */
static double pt_jacobi2d5(const geom_t* g, const void* in, const double* c,
                           int64_t j, int64_t i) {
    const int dt = g->dt;
    return c[0] * rd(in, dt, I2(g, j, i))
         + c[1] * (rd(in, dt, I2(g, j, i - 1)) + rd(in, dt, I2(g, j - 1, i))
                   + rd(in, dt, I2(g, j, i + 1)) + rd(in, dt, I2(g, j + 1, i)));
}

/* gaussblur5x5 — Table 1 "gaussblur ... 20 / 25": 25 loads,
 * a 5x5 neighbourhood.  Reading R4: correlation with weights w[dj][di],
 *   acc = 0; for dj=-2..2: for di=-2..2: acc = acc + w[dj+2][di+2]*in[j+dj][i+di] */
static double pt_gaussblur(const geom_t* g, const void* in, const double* w,
                           int64_t j, int64_t i) {
    double acc = 0.0;
    for (int dj = -2; dj <= 2; ++dj)
        for (int di = -2; di <= 2; ++di)
            acc = acc + w[(dj + 2) * 5 + (di + 2)] * rd(in, g->dt, I2(g, j + dj, i + di));
    return acc;
}

/* gameoflife — Table 1 "gameoflife ... 6 / 9": 9 loads
 * (8 neighbours + centre).  Reading R5: Conway B3/S23 on int cells,
 *   n = sum of the 8 neighbours; out = (n==3 || (n==2 && c==1)) ? 1 : 0 */
static int32_t pt_gameoflife(const geom_t* g, const int32_t* in, int64_t j, int64_t i) {
    int32_t n = in[I2(g, j - 1, i - 1)] + in[I2(g, j - 1, i)] + in[I2(g, j - 1, i + 1)]
              + in[I2(g, j, i - 1)] + in[I2(g, j, i + 1)]
              + in[I2(g, j + 1, i - 1)] + in[I2(g, j + 1, i)] + in[I2(g, j + 1, i + 1)];
    int32_t c = in[I2(g, j, i)];
    return (n == 3 || (n == 2 && c == 1)) ? 1 : 0;
}

/* ----------------------------------------------- 3-D point definitions */

/* laplacian3d7 / jacobi3d7 — Table 1 "laplacian ... 2 / 7":
 * 7 loads.  Reading R6:
 *   out = a*in[k][j][i] + b*(in[k][j][i+1] + in[k][j][i-1] + in[k][j+1][i]
 *                            + in[k][j-1][i] + in[k+1][j][i] + in[k-1][j][i])
 * jacobi3d7 is the same formula with Jacobi weights (reading R7). */
static double pt_lap7(const geom_t* g, const void* in, const double* c,
                      int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    return c[0] * rd(in, dt, I3(g, k, j, i))
         + c[1] * (rd(in, dt, I3(g, k, j, i + 1)) + rd(in, dt, I3(g, k, j, i - 1))
                   + rd(in, dt, I3(g, k, j + 1, i)) + rd(in, dt, I3(g, k, j - 1, i))
                   + rd(in, dt, I3(g, k + 1, j, i)) + rd(in, dt, I3(g, k - 1, j, i)));
}

/* wave13pt — Table 1 "wave13pt ... 4 / 14": 13 taps of the
 * current time level + 1 of the previous.  Reading R8 (leapfrog):
 *   next = m0*cur[c]
 *        + m1*(cur[i+1]+cur[i-1]+cur[j+1]+cur[j-1]+cur[k+1]+cur[k-1])
 *        + m2*(cur[i+2]+cur[i-2]+cur[j+2]+cur[j-2]+cur[k+2]+cur[k-2])
 *        - prev[c]                                                      */
static double pt_wave13(const geom_t* g, const void* prev, const void* cur,
                        const double* m, int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    return m[0] * rd(cur, dt, I3(g, k, j, i))
         + m[1] * (rd(cur, dt, I3(g, k, j, i + 1)) + rd(cur, dt, I3(g, k, j, i - 1))
                   + rd(cur, dt, I3(g, k, j + 1, i)) + rd(cur, dt, I3(g, k, j - 1, i))
                   + rd(cur, dt, I3(g, k + 1, j, i)) + rd(cur, dt, I3(g, k - 1, j, i)))
         + m[2] * (rd(cur, dt, I3(g, k, j, i + 2)) + rd(cur, dt, I3(g, k, j, i - 2))
                   + rd(cur, dt, I3(g, k, j + 2, i)) + rd(cur, dt, I3(g, k, j - 2, i))
                   + rd(cur, dt, I3(g, k + 2, j, i)) + rd(cur, dt, I3(g, k - 2, j, i)))
         - rd(prev, dt, I3(g, k, j, i));
}

/* divergence — Table 1 "divergence ... 1 / 6": 6 loads
 * from three arrays.  Reading R9 (central differences):
 *   out = ax*(u[k][j][i+1]-u[k][j][i-1]) + ay*(v[k][j+1][i]-v[k][j-1][i])
 *       + az*(w[k+1][j][i]-w[k-1][j][i])                               */
static double pt_divergence(const geom_t* g, const void* u, const void* v,
                            const void* w, const double* a, int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    return a[0] * (rd(u, dt, I3(g, k, j, i + 1)) - rd(u, dt, I3(g, k, j, i - 1)))
         + a[1] * (rd(v, dt, I3(g, k, j + 1, i)) - rd(v, dt, I3(g, k, j - 1, i)))
         + a[2] * (rd(w, dt, I3(g, k + 1, j, i)) - rd(w, dt, I3(g, k - 1, j, i)));
}

/* gradient — Table 1 "gradient ... 1 / 6": 6 loads from one
 * array, three outputs.  Reading R10:
 *   gx = ax*(u[i+1]-u[i-1]); gy = ay*(u[j+1]-u[j-1]); gz = az*(u[k+1]-u[k-1]) */
static void pt_gradient(const geom_t* g, const void* u, const double* a,
                        int64_t k, int64_t j, int64_t i, double* gx, double* gy, double* gz) {
    const int dt = g->dt;
    *gx = a[0] * (rd(u, dt, I3(g, k, j, i + 1)) - rd(u, dt, I3(g, k, j, i - 1)));
    *gy = a[1] * (rd(u, dt, I3(g, k, j + 1, i)) - rd(u, dt, I3(g, k, j - 1, i)));
    *gz = a[2] * (rd(u, dt, I3(g, k + 1, j, i)) - rd(u, dt, I3(g, k - 1, j, i)));
}

/* tricubic — Table 1 "tricubic ... 48 / 67": 64 taps of a
 * 4x4x4 neighbourhood + 3 per-point offsets.  Reading R11: cubic Lagrange
 * interpolation on nodes {-1,0,1,2} at offset t in each axis,
 *   L(t) = { -t(t-1)(t-2)/6, (t+1)(t-1)(t-2)/2, -(t+1)t(t-2)/2, (t+1)t(t-1)/6 }
 *   g = sum_c wz[c] * ( sum_b wy[b] * ( sum_a wx[a] * f[k+c-1][j+b-1][i+a-1] ) )
 * each sum in index order starting from its first product.             */
static void lagrange4(double t, double L[4]) {
    L[0] = -t * (t - 1.0) * (t - 2.0) / 6.0;
    L[1] = (t + 1.0) * (t - 1.0) * (t - 2.0) / 2.0;
    L[2] = -(t + 1.0) * t * (t - 2.0) / 2.0;
    L[3] = (t + 1.0) * t * (t - 1.0) / 6.0;
}
static double pt_tricubic(const geom_t* g, const void* f, const void* X, const void* Y,
                          const void* Z, int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    double wx[4], wy[4], wz[4];
    lagrange4(rd(X, dt, I3(g, k, j, i)), wx);
    lagrange4(rd(Y, dt, I3(g, k, j, i)), wy);
    lagrange4(rd(Z, dt, I3(g, k, j, i)), wz);
    double sc = 0.0;
    for (int c = 0; c < 4; ++c) {
        double sb = 0.0;
        for (int b = 0; b < 4; ++b) {
            double sa = wx[0] * rd(f, dt, I3(g, k + c - 1, j + b - 1, i - 1));
            for (int a = 1; a < 4; ++a)
                sa = sa + wx[a] * rd(f, dt, I3(g, k + c - 1, j + b - 1, i + a - 1));
            sb = (b == 0) ? wy[0] * sa : sb + wy[b] * sa;
        }
        sc = (c == 0) ? wz[0] * sb : sc + wz[c] * sb;
    }
    return sc;
}

/* tricubic2 — Table 1 "tricubic2 ... 48 / 67", the same
 * 64 + 3 loads and the same 48 shuffles as tricubic.  Reading R19: the same
 * interpolation (cubic Lagrange on nodes {-1,0,1,2}, R11) written as the
 * fully expanded 64-term sum, each term's weight the product of its three
 * 1-D weights:
 *   g = sum_c sum_b sum_a ((wx[a]*wy[b])*wz[c]) * f[k+c-1][j+b-1][i+a-1]
 * one running sum, c outer, a inner, starting from the first product.     */
static double pt_tricubic2(const geom_t* g, const void* f, const void* X, const void* Y,
                           const void* Z, int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    double wx[4], wy[4], wz[4];
    lagrange4(rd(X, dt, I3(g, k, j, i)), wx);
    lagrange4(rd(Y, dt, I3(g, k, j, i)), wy);
    lagrange4(rd(Z, dt, I3(g, k, j, i)), wz);
    double s = 0.0;
    for (int c = 0; c < 4; ++c)
        for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a) {
                const double t = ((wx[a] * wy[b]) * wz[c]) * rd(f, dt, I3(g, k + c - 1, j + b - 1, i + a - 1));
                s = (a == 0 && b == 0 && c == 0) ? t : s + t;
            }
    return s;
}

/* uxx1 — Table 1 "uxx1 ... 3 / 17, delta 2.00" (512x512x1024,
 * PAPER.md:645-646).  Reading R20: the velocity update u1 of a 4th-order
 * staggered-grid elastic wave code, one output from five arrays
 * (u1, d1, xx, xy, xz), lo = 2, hi = 1 per axis:
 *   d   = 0.25*(d1[k][j][i] + d1[k][j-1][i] + d1[k-1][j][i] + d1[k-1][j-1][i])
 *   out = u1[k][j][i] + (dth/d) * ( c1*(xx[i]-xx[i-1] + xy[j]-xy[j-1] + xz[k]-xz[k-1])
 *                                 + c2*(xx[i+1]-xx[i-2] + xy[j+1]-xy[j-2] + xz[k+1]-xz[k-2]) )
 * (xx taps along x, xy along y, xz along z, at the point otherwise).
 * Loads: u1 1 + d1 4 + xx 4 + xy 4 + xz 4 = 17; only xx's four taps share
 * an x-row: 3 shuffles of delta 1, 2, 3 from the x-end (R1): 2.00.        */
static double pt_uxx1(const geom_t* g, const void* const* in, const double* c,
                      int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    const void *u1 = in[0], *d1 = in[1], *xx = in[2], *xy = in[3], *xz = in[4];
    const double d = 0.25 * (rd(d1, dt, I3(g, k, j, i)) + rd(d1, dt, I3(g, k, j - 1, i))
                             + rd(d1, dt, I3(g, k - 1, j, i)) + rd(d1, dt, I3(g, k - 1, j - 1, i)));
    const double s1 = rd(xx, dt, I3(g, k, j, i)) - rd(xx, dt, I3(g, k, j, i - 1))
                    + rd(xy, dt, I3(g, k, j, i)) - rd(xy, dt, I3(g, k, j - 1, i))
                    + rd(xz, dt, I3(g, k, j, i)) - rd(xz, dt, I3(g, k - 1, j, i));
    const double s2 = rd(xx, dt, I3(g, k, j, i + 1)) - rd(xx, dt, I3(g, k, j, i - 2))
                    + rd(xy, dt, I3(g, k, j + 1, i)) - rd(xy, dt, I3(g, k, j - 2, i))
                    + rd(xz, dt, I3(g, k + 1, j, i)) - rd(xz, dt, I3(g, k - 2, j, i));
    return rd(u1, dt, I3(g, k, j, i)) + (c[0] / d) * (c[1] * s1 + c[2] * s2);
}

/* lapgsrb — Table 1 "lapgsrb ... 12 / 25, delta 1.83", the
 * red-black Gauss-Seidel smoother of the 3-D Laplace operator ("lap" +
 * "gsrb").  Reading R21: one full red-black iteration (red half-sweep, then
 * black half-sweep reading the new red values) as one out-of-place
 * point-wise pass, w the Gauss-Seidel weight (1/6 by default):
 *   red(p)  = (i+j+k) even
 *   nb6(q)  = u[q-x] + u[q+x] + u[q-y] + u[q+y] + u[q-z] + u[q+z]   (that order)
 *   r(q)    = w*nb6(q) if q is an interior red point, else u[q]  (the boundary ring is held)
 *   out(p)  = red(p) ? r(p) : w*(r(p-x) + r(p+x) + r(p-y) + r(p+y) + r(p-z) + r(p+z))
 * A black point's six neighbours are red; each new red value is recomputed
 * from the old field, so the loads of one point are the 25 points at L1
 * distance <= 2 (6 for a red point, 19 for a black one; the lanes of a warp
 * alternate between the two branches: divergent).  Their x-rows give 12
 * shuffles of total delta 22 from the x-end (R1): 1.83.  The boundary ring
 * is 1 wide: reads stay inside the grid because r of a ring point is u.   */
static int lap_interior(const geom_t* g, int64_t k, int64_t j, int64_t i) {
    return i >= 1 && i < g->nx - 1 && j >= 1 && j < g->ny - 1 && k >= 1 && k < g->nz - 1;
}
static double lap_nb6(const geom_t* g, const void* u, int64_t k, int64_t j, int64_t i) {
    const int dt = g->dt;
    return rd(u, dt, I3(g, k, j, i - 1)) + rd(u, dt, I3(g, k, j, i + 1))
         + rd(u, dt, I3(g, k, j - 1, i)) + rd(u, dt, I3(g, k, j + 1, i))
         + rd(u, dt, I3(g, k - 1, j, i)) + rd(u, dt, I3(g, k + 1, j, i));
}
static double lap_red(const geom_t* g, const void* u, double w, int64_t k, int64_t j, int64_t i) {
    if (lap_interior(g, k, j, i) && ((i + j + k) & 1) == 0) return w * lap_nb6(g, u, k, j, i);
    return rd(u, g->dt, I3(g, k, j, i));
}
static double pt_lapgsrb(const geom_t* g, const void* u, const double* c,
                         int64_t k, int64_t j, int64_t i) {
    const double w = c[0];
    if (((i + j + k) & 1) == 0) return lap_red(g, u, w, k, j, i);
    return w * (lap_red(g, u, w, k, j, i - 1) + lap_red(g, u, w, k, j, i + 1)
                + lap_red(g, u, w, k, j - 1, i) + lap_red(g, u, w, k, j + 1, i)
                + lap_red(g, u, w, k - 1, j, i) + lap_red(g, u, w, k + 1, j, i));
}

/* whispering — Table 1 "whispering ... 6 / 19, delta 0.83" (
 * 2-D, "more buffers are allocated", 8192x16384).
 * Reading R22: one leapfrog step of the 2-D TM-mode Yee scheme (FDTD) of a
 * whispering-gallery resonator — per-cell material arrays carry the
 * dielectric (cb) and the absorbing layer (dax, dbx, day, dby) — with the
 * magnetic half step fused into the electric one: the two neighbouring H
 * values the Ez update needs are recomputed from the old fields.
 * in = (Hx, Hy, Ez, dax, dbx, day, dby, cb), out = (Hx', Hy', Ez'):
 *   hx(q) = dax[q]*Hx[q] - dbx[q]*(Ez[q+y] - Ez[q])
 *   hy(q) = day[q]*Hy[q] + dby[q]*(Ez[q+x] - Ez[q])
 *   Hx'(p) = hx(p);  Hy'(p) = hy(p)
 *   Ez'(p) = Ez[p] + cb[p]*((hy(p) - hy(p-x)) - (hx(p) - hx(p-y)))
 * 18 distinct taps; Ez[p] is loaded again for Ez' after the stores of Hx'
 * and Hy' (the N=0 reuse): 19 loads, 6 shuffles of total delta 5.        */
static double wh_hx(const geom_t* g, const void* const* in, int64_t j, int64_t i) {
    const int dt = g->dt;
    return rd(in[3], dt, I2(g, j, i)) * rd(in[0], dt, I2(g, j, i))
         - rd(in[4], dt, I2(g, j, i)) * (rd(in[2], dt, I2(g, j + 1, i)) - rd(in[2], dt, I2(g, j, i)));
}
static double wh_hy(const geom_t* g, const void* const* in, int64_t j, int64_t i) {
    const int dt = g->dt;
    return rd(in[5], dt, I2(g, j, i)) * rd(in[1], dt, I2(g, j, i))
         + rd(in[6], dt, I2(g, j, i)) * (rd(in[2], dt, I2(g, j, i + 1)) - rd(in[2], dt, I2(g, j, i)));
}
static void pt_whispering(const geom_t* g, const void* const* in, int64_t j, int64_t i,
                          double* hx, double* hy, double* ez) {
    const int dt = g->dt;
    *hx = wh_hx(g, in, j, i);
    *hy = wh_hy(g, in, j, i);
    *ez = rd(in[2], dt, I2(g, j, i))
        + rd(in[7], dt, I2(g, j, i)) * ((*hy - wh_hy(g, in, j, i - 1)) - (*hx - wh_hx(g, in, j - 1, i)));
}

/* ------------------------------------------------------------- driver */
static int check(const kind_t* k, int dt, int ndims, const int64_t* dims, int ncoeffs) {
    if (!k) return fail("unknown kind");
    if (dt == DT_BAD) return fail("unknown dtype");
    if (dt == DT_I32 && !k->allow_i) return fail("dtype not allowed for kind");
    if (dt != DT_I32 && !k->allow_f) return fail("dtype not allowed for kind");
    if (ndims != k->ndims) return fail("wrong ndims");
    if (ncoeffs != 0 && ncoeffs != k->ncoeffs) return fail("wrong ncoeffs");
    for (int d = 0; d < ndims; ++d)
        if (dims[d] < k->lo + k->hi + 1) return fail("axis too small for one interior point");
    return 0;
}

int oracle_step(const char* kind, const char* dtype, int ndims, const int64_t* dims,
                const double* coeffs, int ncoeffs, const void* const* in,
                void* const* out, int nthreads) {
    const kind_t* k = find_kind(kind);
    const int dt = parse_dtype(dtype);
    if (check(k, dt, ndims, dims, ncoeffs)) return -1;
    double c[32];
    if (ncoeffs == 0) oracle_default_coeffs(kind, c, 32);
    else memcpy(c, coeffs, sizeof(double) * (size_t)ncoeffs);
    geom_t g = {dims[0], dims[1], ndims == 3 ? dims[2] : 1, dt};
    const int lo = k->lo, hi = k->hi;
    if (nthreads <= 0) nthreads = 1;
    (void)nthreads;
    const int kid = (int)(k - KINDS);   /* index into KINDS[] */

    if (k->ndims == 2) {
        #pragma omp parallel for num_threads(nthreads) schedule(static)
        for (int64_t j = lo; j < g.ny - hi; ++j)
            for (int64_t i = lo; i < g.nx - hi; ++i) {
                const int64_t o = I2(&g, j, i);
                switch (kid) {
                case 0: wr(out[0], dt, o, pt_jacobi2d5(&g, in[0], c, j, i)); break;
                case 1: wr(out[0], dt, o, pt_jacobi2d9(&g, in[0], c, j, i)); break;
                case 2: wr(out[0], dt, o, pt_gaussblur(&g, in[0], c, j, i)); break;
                case 3: ((int32_t*)out[0])[o] = pt_gameoflife(&g, (const int32_t*)in[0], j, i); break;
                default: {          /* whispering: out = (Hx', Hy', Ez') */
                    double hx, hy, ez;
                    pt_whispering(&g, in, j, i, &hx, &hy, &ez);
                    wr(out[0], dt, o, hx);
                    wr(out[1], dt, o, hy);
                    wr(out[2], dt, o, ez);
                }
                }
            }
        return 0;
    }
    #pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t kk = lo; kk < g.nz - hi; ++kk)
        for (int64_t j = lo; j < g.ny - hi; ++j)
            for (int64_t i = lo; i < g.nx - hi; ++i) {
                const int64_t o = I3(&g, kk, j, i);
                switch (kid) {
                case 4: case 5:      /* laplacian3d7, jacobi3d7 */
                    wr(out[0], dt, o, pt_lap7(&g, in[0], c, kk, j, i)); break;
                case 6:              /* wave13pt: in = (prev, cur) */
                    wr(out[0], dt, o, pt_wave13(&g, in[0], in[1], c, kk, j, i)); break;
                case 7:              /* divergence: in = (u, v, w) */
                    wr(out[0], dt, o, pt_divergence(&g, in[0], in[1], in[2], c, kk, j, i)); break;
                case 8: {            /* gradient: out = (gx, gy, gz) */
                    double gx, gy, gz;
                    pt_gradient(&g, in[0], c, kk, j, i, &gx, &gy, &gz);
                    wr(out[0], dt, o, gx);
                    wr(out[1], dt, o, gy);
                    wr(out[2], dt, o, gz);
                    break;
                }
                case 9:              /* tricubic: in = (f, X, Y, Z) */
                    wr(out[0], dt, o, pt_tricubic(&g, in[0], in[1], in[2], in[3], kk, j, i)); break;
                case 10:             /* tricubic2: the expanded 64-term form */
                    wr(out[0], dt, o, pt_tricubic2(&g, in[0], in[1], in[2], in[3], kk, j, i)); break;
                case 11:             /* uxx1: in = (u1, d1, xx, xy, xz) */
                    wr(out[0], dt, o, pt_uxx1(&g, in, c, kk, j, i)); break;
                default:             /* lapgsrb */
                    wr(out[0], dt, o, pt_lapgsrb(&g, in[0], c, kk, j, i));
                }
            }
    return 0;
}

/* Copy every non-interior point of src into dst (the Dirichlet ring). */
static void copy_ring(const geom_t* g, int ndims, int lo, int hi, const void* src, void* dst) {
    const size_t es = dt_size(g->dt);
    const int64_t nz = ndims == 3 ? g->nz : 1;
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < g->ny; ++j)
            for (int64_t i = 0; i < g->nx; ++i) {
                int interior = i >= lo && i < g->nx - hi && j >= lo && j < g->ny - hi;
                if (ndims == 3) interior = interior && k >= lo && k < nz - hi;
                if (!interior) {
                    const int64_t o = (k * g->ny + j) * g->nx + i;
                    memcpy((char*)dst + o * es, (const char*)src + o * es, es);
                }
            }
}

int oracle_run(const char* kind, const char* dtype, int ndims, const int64_t* dims,
               const double* coeffs, int ncoeffs, void* const* bufs, int n_iters,
               int nthreads, int* result_idx) {
    const kind_t* k = find_kind(kind);
    const int dt = parse_dtype(dtype);
    if (check(k, dt, ndims, dims, ncoeffs)) return -1;
    if (n_iters < 0) return fail("n_iters < 0");
    geom_t g = {dims[0], dims[1], ndims == 3 ? dims[2] : 1, dt};

    if (k->iterable == 1) {            /* ping-pong bufs[0] <-> bufs[1] */
        copy_ring(&g, ndims, k->lo, k->hi, bufs[0], bufs[1]);
        int cur = 0;
        for (int it = 0; it < n_iters; ++it) {
            const void* in[1] = {bufs[cur]};
            void* out[1] = {bufs[1 - cur]};
            if (oracle_step(kind, dtype, ndims, dims, coeffs, ncoeffs, in, out, nthreads)) return -1;
            cur = 1 - cur;
        }
        if (result_idx) *result_idx = cur;
        return 0;
    }
    if (k->iterable == 2) {            /* wave13pt: bufs = (prev, cur, next) */
        copy_ring(&g, ndims, k->lo, k->hi, bufs[1], bufs[0]);
        copy_ring(&g, ndims, k->lo, k->hi, bufs[1], bufs[2]);
        int p = 0, c = 1, nx = 2;
        for (int it = 0; it < n_iters; ++it) {
            const void* in[2] = {bufs[p], bufs[c]};
            void* out[1] = {bufs[nx]};
            if (oracle_step(kind, dtype, ndims, dims, coeffs, ncoeffs, in, out, nthreads)) return -1;
            const int t = p; p = c; c = nx; nx = t;   /* (prev,cur,next) <- (cur,next,prev) */
        }
        if (result_idx) *result_idx = c;
        return 0;
    }
    /* divergence / gradient / tricubic / tricubic2 / uxx1 / whispering: re-apply the same step */
    const void* in[8];
    void* out[3];
    for (int a = 0; a < k->n_in; ++a) in[a] = bufs[a];
    for (int a = 0; a < k->n_out; ++a) out[a] = bufs[k->n_in + a];
    for (int it = 0; it < n_iters; ++it)
        if (oracle_step(kind, dtype, ndims, dims, coeffs, ncoeffs, in, out, nthreads)) return -1;
    if (result_idx) *result_idx = k->n_in;
    return 0;
}
