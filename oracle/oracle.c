/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct float64 CPU implementation of the one
 * computation this repository accelerates.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_1405_7470_b200/) never links, imports or executes it,
 * and this file shares no code, header, table or helper with the CUDA side.
 *
 * What it computes (section 2.1, the reduction example;
 * and, at the end of this file, Table 1's saxpy, and 3D Coulomb
 * potential):
 *
 *     c[i,j] = sum(k, a[i,k]*b[k,j])
 *
 * over the loop domain { [i,j,k] : 0<=i<M, 0<=j<N, 0<=k<K }  (P:211-224,
 * section 2.1: a box over the inames i, j, k with parameters M, N, K).
 *
 *  - Inputs are fp32 (section 2.2: type inference, single precision
 *    in -> single precision out).  Each product of two fp32 values is exact in
 *    float64 (24+24 <= 53 significant bits), so the only rounding is in the
 *    float64 sum; k is summed in ascending order (the lexicographic order of
 *    SPEC.md's reference_run).
 *  - Layout semantics follow the per-axis stride tags (P:278-280, P:313-315,
 *    P:594-601): row-major X(r,c) = X[r*ld + c], column-major X(r,c) = X[r + c*ld].
 *  - K == 0 gives 0 (the identity of `sum`); M == 0 or N == 0 is
 *    an empty domain and writes nothing.
 *  - It also returns D[i,j] = sum_k |a[i,k]| |b[k,j]|, the denominator of the
 *    normalised error of the parity contract (BASELINE.json north_star).
 *
 * Outputs are always packed row-major float64 arrays (result row i - row0 at
 * offset (i - row0)*N).  Parallelism is over i only (OpenMP), so each element's
 * summation order is fixed and results are bitwise reproducible for any thread
 * count.  Pins: tests/test_oracle.py (exact rational brute force, closed forms,
 * worked examples, library cross-check) -- see DESIGN.md "Oracle pins".
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_ROW_MAJOR 0
#define ORACLE_COL_MAJOR 1

/* X(r, c) for a matrix stored with `layout` and leading dimension `ld`. */
static inline double at(const float *X, int64_t ld, int layout, int64_t r, int64_t c)
{
    return (double)(layout == ORACLE_ROW_MAJOR ? X[r * ld + c] : X[r + c * ld]);
}

static int bad_args(int64_t M, int64_t N, int64_t K, int la, int lb)
{
    if (M < 0 || N < 0 || K < 0) return 1;
    if ((la != ORACLE_ROW_MAJOR && la != ORACLE_COL_MAJOR) ||
        (lb != ORACLE_ROW_MAJOR && lb != ORACLE_COL_MAJOR)) return 1;
    return 0;
}

/* Rows [row0, row1) of C = A*B and of D = |A|*|B|.  Returns 0, or -1 on bad
 * arguments.  nthreads <= 0 uses the OpenMP default. */
int lpy_oracle_gemm_rows_f64(int64_t M, int64_t N, int64_t K,
                             const float *A, int64_t lda, int la,
                             const float *B, int64_t ldb, int lb,
                             int64_t row0, int64_t row1,
                             double *C, double *D, int nthreads)
{
    if (bad_args(M, N, K, la, lb) || row0 < 0 || row1 > M || row0 > row1) return -1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t i = row0; i < row1; ++i) {
        double *c = C + (i - row0) * N;
        double *d = D ? D + (i - row0) * N : NULL;
        for (int64_t j = 0; j < N; ++j) {
            c[j] = 0.0;                       /* sum identity */
            if (d) d[j] = 0.0;
        }
        for (int64_t k = 0; k < K; ++k) {     /* k ascending */
            const double a = at(A, lda, la, i, k);
            for (int64_t j = 0; j < N; ++j) {
                const double b = at(B, ldb, lb, k, j);
                c[j] += a * b;                /* a*b exact in float64 */
                if (d) d[j] += fabs(a) * fabs(b);
            }
        }
    }
    (void)nthreads;
    return 0;
}

/* The full product: rows [0, M). */
int lpy_oracle_gemm_f64(int64_t M, int64_t N, int64_t K,
                        const float *A, int64_t lda, int la,
                        const float *B, int64_t ldb, int lb,
                        double *C, double *D, int nthreads)
{
    return lpy_oracle_gemm_rows_f64(M, N, K, A, lda, la, B, ldb, lb, 0, M, C, D, nthreads);
}

/* Selected elements (ii[e], jj[e]), e < count: the same k-ascending float64 sum
 * as above, so each value is bitwise identical to the full product's. */
int lpy_oracle_gemm_elems_f64(int64_t M, int64_t N, int64_t K,
                              const float *A, int64_t lda, int la,
                              const float *B, int64_t ldb, int lb,
                              int64_t count, const int64_t *ii, const int64_t *jj,
                              double *C, double *D, int nthreads)
{
    if (bad_args(M, N, K, la, lb) || count < 0) return -1;
    for (int64_t e = 0; e < count; ++e)
        if (ii[e] < 0 || ii[e] >= M || jj[e] < 0 || jj[e] >= N) return -1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t e = 0; e < count; ++e) {
        double c = 0.0, d = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            const double a = at(A, lda, la, ii[e], k);
            const double b = at(B, ldb, lb, k, jj[e]);
            c += a * b;
            d += fabs(a) * fabs(b);
        }
        C[e] = c;
        if (D) D[e] = d;
    }
    (void)nthreads;
    return 0;
}

/* ------------------------------------------------------------------ saxpy
 * Table 1's "saxpy" row (section 3): y := alpha * x + y.
 * out[i] = (double)alpha * (double)x[i*incx] + (double)y[i*incy] for i < n,
 * in float64: the product of two fp32 values is exact in float64 and the sum
 * rounds once (relative error <= 2^-53), so `out` is the exact value of
 * alpha*x_i + y_i for the parity contract (the fp32 result must be its
 * round-to-nearest, reading S1).  x and y are only read; returns 0,
 * or -1 on bad arguments (n < 0, inc < 1). */
int lpy_oracle_saxpy_f64(int64_t n, float alpha, const float *x, int64_t incx,
                         const float *y, int64_t incy, double *out, int nthreads)
{
    if (n < 0 || incx < 1 || incy < 1) return -1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < n; ++i)
        out[i] = (double)alpha * (double)x[i * incx] + (double)y[i * incy];
    (void)nthreads;
    return 0;
}

/* ------------------------------------------------------------------ Coulomb
 * Table 1's "3D Coulomb pot." row (section 3): the potential
 * at each target of a set of point charges,
 *
 *     phi[i] = sum_{j : r_ij != 0} q[j] / r_ij,
 *     r_ij   = sqrt((tx_i - sx_j)^2 + (ty_i - sy_j)^2 + (tz_i - sz_j)^2),
 *
 * for i < nt over the sources j < ns, j ascending.  A source at exactly the
 * target's position (r_ij = 0: the target itself when targets == sources)
 * contributes nothing (reading C1).  Target i's coordinates are
 * t[i*ldt + 0..2], source j's s[j*lds + 0..2], its charge q[j] (fp32 in).
 * Everything is float64: coordinate differences of fp32 values are exact in
 * float64, the rest rounds at 2^-53 per operation, so phi is exact to far
 * below the GPU tolerance.  Also returns D[i] = sum_j |q[j]| / r_ij, the
 * normaliser of the parity metric |phi - phi_ref| / D.  Parallel over i only;
 * returns 0, or -1 on bad arguments. */
int lpy_oracle_coulomb_f64(int64_t nt, const float *t, int64_t ldt,
                           int64_t ns, const float *s, int64_t lds, const float *q,
                           double *phi, double *D, int nthreads)
{
    if (nt < 0 || ns < 0 || ldt < 3 || lds < 3) return -1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < nt; ++i) {
        const double x = t[i * ldt], y = t[i * ldt + 1], z = t[i * ldt + 2];
        double acc = 0.0, dacc = 0.0;
        for (int64_t j = 0; j < ns; ++j) {
            const double dx = x - (double)s[j * lds];
            const double dy = y - (double)s[j * lds + 1];
            const double dz = z - (double)s[j * lds + 2];
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            if (r == 0.0) continue;          /* coincident: excluded (reading C1) */
            acc += (double)q[j] / r;
            dacc += fabs((double)q[j]) / r;
        }
        phi[i] = acc;
        if (D) D[i] = dacc;
    }
    (void)nthreads;
    return 0;
}

/* Number of OpenMP threads a call with nthreads <= 0 would use. */
int lpy_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
