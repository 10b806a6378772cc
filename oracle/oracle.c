/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of the batched GEMM of
 * Jhurani & Mullowney, arXiv:1304.7053.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1304_7053_b200/) never includes, links or calls it,
 * and this file includes nothing from the product tree.
 *
 * What it computes (§2 Eq. (1)):
 *     C^p <- alpha * op(A^p) * op(B^p) + beta * C^p,   p = 1..N independently,
 * with op(X) in {X, X^T, X^*} chosen independently for A and B (PAPER.md:240-243,
 * 256-258), C m x n, op(A) m x k, op(B) k x n, for the four
 * scalar types S/D/C/Z.
 *
 * Indexing: the (i,j) entry of the p-th matrix is X[i + ldx*j + ldx2*p], in
 * units of scalar elements, not bytes (§5).  The pointer
 * variant uses Xarray[p] + i + ldx*j (cuBLAS-like interface, PAPER.md:273-286,
 * TGEMM_multi_nounif).
 *
 * Order of operations (rows 1-4, 16):
 *   x = sum over l = 0..k-1 in ascending order, in the working precision,
 *       no fused multiply-add (built with -ffp-contract=off);
 *   complex products by the textbook 4-multiply/2-add formula, "3M" not used
 *       (PAPER.md:570-572);
 *   then y = a*x + b*y (the paper's axpby functor), or
 *   y = a*x without reading y when beta == 0 (BLAS semantics; the paper's
 *   a1b0 functor never reads C);
 *   alpha == 0 or k == 0: A and B are never read, C <- beta*C;
 *   quick return (C untouched) when m == 0, n == 0, batch == 0, or
 *   (alpha == 0 or k == 0) and beta == 1.
 *
 * Return codes are the boundary's (include/txgemm.h): 0, or -i when argument i
 * (1-based) is invalid; the validation below is an independent re-implementation
 * of the rules listed in DESIGN.md §Boundary.
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (closed forms, hand cases, library routine, exact rational arithmetic,
 * invariants).  No function is "parity unpinned".
 */
#include <stddef.h>
#include <stdint.h>

typedef struct { float re, im; } o_cfloat;
typedef struct { double re, im; } o_cdouble;

#define O_MAXDIM_REAL 64 /* s, d (reading R14) */
#define O_MAXDIM_CPLX 32 /* c, z */

/* ---------------------------------------------------------------- helpers */

static int op_valid(char c)
{
    return c == 'n' || c == 'N' || c == 't' || c == 'T' || c == 'c' || c == 'C';
}
static int op_is_n(char c) { return c == 'n' || c == 'N'; }
static int op_is_c(char c) { return c == 'c' || c == 'C'; }
static int imax1(int a) { return a > 1 ? a : 1; }

/* Extent in elements of one batch operand: [0, ld2*(batch-1) + ld*(cols-1) + rows). */
static long long extent(int rows, int cols, int ld, long long ld2, int batch)
{
    if (rows <= 0 || cols <= 0 || batch <= 0) return 0;
    return ld2 * (long long)(batch - 1) + (long long)ld * (cols - 1) + rows;
}

static int ranges_overlap(const void *p, long long np, const void *q, long long nq, size_t esz)
{
    if (np <= 0 || nq <= 0) return 0;
    uintptr_t a0 = (uintptr_t)p, a1 = a0 + (uintptr_t)np * esz;
    uintptr_t b0 = (uintptr_t)q, b1 = b0 + (uintptr_t)nq * esz;
    return a0 < b1 && b0 < a1;
}

/*
 * Argument checks, in the order of DESIGN.md §Boundary (argument positions of
 * the strided call; the pointer call's positions in brackets):
 *   transa -1, transb -2, m -3, n -4, k -5 (each in [0,64] for s/d, [0,32] for c/z),
 *   alpha NULL -6,
 *   beta NULL -13 [-11], lda -8, ldb -11 [-10], ldc -15 [-13],
 *   (batch > 1) lda2 < 0 -9, ldb2 < 0 -12, ldc2 < ldc*n -16  (Fig. 1),
 *   batch < 0 -17 [-14], A NULL or misaligned -7, B -10 [-9], C -14 [-12],
 *   (strided) C's extent overlapping A's or B's -14.
 */
static int validate(int ptr, char ta, char tb, int m, int n, int k,
                    const void *alpha, int alpha_is_zero, const void *beta,
                    const void *A, int lda, long long lda2,
                    const void *B, int ldb, long long ldb2,
                    const void *C, int ldc, long long ldc2, int batch, size_t esz,
                    int maxdim)
{
    if (!op_valid(ta)) return -1;
    if (!op_valid(tb)) return -2;
    if (m < 0 || m > maxdim) return -3;
    if (n < 0 || n > maxdim) return -4;
    if (k < 0 || k > maxdim) return -5;
    if (alpha == NULL) return -6;
    if (beta == NULL) return ptr ? -11 : -13;
    int rowsA = op_is_n(ta) ? m : k, colsA = op_is_n(ta) ? k : m;
    int rowsB = op_is_n(tb) ? k : n, colsB = op_is_n(tb) ? n : k;
    if (lda < imax1(rowsA)) return -8;
    if (ldb < imax1(rowsB)) return ptr ? -10 : -11;
    if (ldc < imax1(m)) return ptr ? -13 : -15;
    if (!ptr && batch > 1) {
        if (lda2 < 0) return -9;
        if (ldb2 < 0) return -12;
        if (ldc2 < (long long)ldc * n) return -16;
    }
    if (batch < 0) return ptr ? -14 : -17;
    int work = m > 0 && n > 0 && batch > 0;
    int reads_ab = work && !alpha_is_zero && k > 0;
    /* NULL, or an address that is not a multiple of the element size (pointer
     * arrays: of the pointer size) -- DESIGN.md reading R21 */
    size_t al = ptr ? sizeof(void *) : esz;
    if (reads_ab && (A == NULL || (uintptr_t)A % al != 0)) return -7;
    if (reads_ab && (B == NULL || (uintptr_t)B % al != 0)) return ptr ? -9 : -10;
    if (work && (C == NULL || (uintptr_t)C % al != 0)) return ptr ? -12 : -14;
    if (!ptr && reads_ab) {
        long long ec = extent(m, n, ldc, ldc2, batch);
        if (ranges_overlap(C, ec, A, extent(rowsA, colsA, lda, lda2, batch), esz)) return -14;
        if (ranges_overlap(C, ec, B, extent(rowsB, colsB, ldb, ldb2, batch), esz)) return -14;
    }
    return 0;
}

/* ------------------------------------------------------------ real types */
/*
 * op(A)_{il} = A[i + lda*l] if transa = N, else A[l + lda*i] ('C' == 'T' for
 * real types: conjugation is the identity).
 * op(B)_{lj} = B[l + ldb*j] if transb = N, else B[j + ldb*l].
 */
#define O_REAL_ONE(NAME, T, ACC)                                                     \
static void NAME(char ta, char tb, int m, int n, int k, T a, T b,                    \
                 const T *Ap, int lda, const T *Bp, int ldb, T *Cp, int ldc)         \
{                                                                                    \
    for (int j = 0; j < n; ++j) {                                                    \
        for (int i = 0; i < m; ++i) {                                                \
            ACC x = 0;                                                               \
            if (a != 0) {                                                            \
                for (int l = 0; l < k; ++l) {                                        \
                    ACC u = op_is_n(ta) ? Ap[i + (long long)lda * l]                 \
                                        : Ap[l + (long long)lda * i];                \
                    ACC v = op_is_n(tb) ? Bp[l + (long long)ldb * j]                 \
                                        : Bp[j + (long long)ldb * l];                \
                    x = x + u * v;                                                   \
                }                                                                    \
            }                                                                        \
            T *y = &Cp[i + (long long)ldc * j];                                      \
            if (b == 0) *y = (T)((ACC)a * x);                                        \
            else        *y = (T)((ACC)a * x + (ACC)b * (ACC)(*y));                   \
        }                                                                            \
    }                                                                                \
}

O_REAL_ONE(one_s, float, float)
O_REAL_ONE(one_d, double, double)

#define O_REAL_API(SUF, T)                                                              \
int oracle_gemm_batched_##SUF(char ta, char tb, int m, int n, int k, const T *alpha,    \
                              const T *A, int lda, long long lda2,                      \
                              const T *B, int ldb, long long ldb2, const T *beta,       \
                              T *C, int ldc, long long ldc2, int batch)                 \
{                                                                                       \
    int rc = validate(0, ta, tb, m, n, k, alpha, alpha && *alpha == 0, beta, A, lda,    \
                      lda2, B, ldb, ldb2, C, ldc, ldc2, batch, sizeof(T), O_MAXDIM_REAL);              \
    if (rc) return rc;                                                                  \
    T a = *alpha, b = *beta;                                                            \
    if (m == 0 || n == 0 || batch == 0 || ((a == 0 || k == 0) && b == 1)) return 0;     \
    if (k == 0) a = 0; /* empty sum: x = 0, A and B not read */                         \
    for (int p = 0; p < batch; ++p)                                                     \
        one_##SUF(ta, tb, m, n, k, a, b, A + lda2 * p, lda, B + ldb2 * p, ldb,          \
                  C + ldc2 * p, ldc);                                                   \
    return 0;                                                                           \
}                                                                                       \
int oracle_gemm_batched_ptr_##SUF(char ta, char tb, int m, int n, int k, const T *alpha,\
                                  const T *const *Aarray, int lda,                      \
                                  const T *const *Barray, int ldb, const T *beta,       \
                                  T *const *Carray, int ldc, int batch)                 \
{                                                                                       \
    int rc = validate(1, ta, tb, m, n, k, alpha, alpha && *alpha == 0, beta, Aarray,    \
                      lda, 0, Barray, ldb, 0, Carray, ldc, 0, batch, sizeof(T), O_MAXDIM_REAL);        \
    if (rc) return rc;                                                                  \
    T a = *alpha, b = *beta;                                                            \
    if (m == 0 || n == 0 || batch == 0 || ((a == 0 || k == 0) && b == 1)) return 0;     \
    if (k == 0) a = 0;                                                                  \
    for (int p = 0; p < batch; ++p)                                                     \
        one_##SUF(ta, tb, m, n, k, a, b, a != 0 ? Aarray[p] : NULL, lda,                \
                  a != 0 ? Barray[p] : NULL, ldb, Carray[p], ldc);                      \
    return 0;                                                                           \
}

O_REAL_API(s, float)
O_REAL_API(d, double)

/* --------------------------------------------------------- complex types */
/*
 * op(A)_{il} as for real types, conjugated when transa = 'C' (the paper's
 * conjugate functor {a.x, -a.y}).  Complex product by the
 * 4-multiply/2-add formula:
 *     (ur + i ui)(vr + i vi) = (ur*vr - ui*vi) + i (ur*vi + ui*vr).
 */
#define O_CPLX_ONE(NAME, CT, ACC)                                                    \
static void NAME(char ta, char tb, int m, int n, int k, CT a, CT b,                  \
                 const CT *Ap, int lda, const CT *Bp, int ldb, CT *Cp, int ldc)      \
{                                                                                    \
    int a_nonzero = !(a.re == 0 && a.im == 0);                                       \
    int b_zero = (b.re == 0 && b.im == 0);                                           \
    for (int j = 0; j < n; ++j) {                                                    \
        for (int i = 0; i < m; ++i) {                                                \
            ACC xr = 0, xi = 0;                                                      \
            if (a_nonzero) {                                                         \
                for (int l = 0; l < k; ++l) {                                        \
                    CT u = op_is_n(ta) ? Ap[i + (long long)lda * l]                  \
                                       : Ap[l + (long long)lda * i];                 \
                    CT v = op_is_n(tb) ? Bp[l + (long long)ldb * j]                  \
                                       : Bp[j + (long long)ldb * l];                 \
                    ACC ur = u.re, ui = op_is_c(ta) ? -(ACC)u.im : (ACC)u.im;        \
                    ACC vr = v.re, vi = op_is_c(tb) ? -(ACC)v.im : (ACC)v.im;        \
                    ACC pr = ur * vr - ui * vi;                                      \
                    ACC pi = ur * vi + ui * vr;                                      \
                    xr = xr + pr;                                                    \
                    xi = xi + pi;                                                    \
                }                                                                    \
            }                                                                        \
            CT *y = &Cp[i + (long long)ldc * j];                                     \
            ACC ar = a.re, ai = a.im;                                                \
            ACC zr = ar * xr - ai * xi; /* a*x */                                    \
            ACC zi = ar * xi + ai * xr;                                              \
            if (!b_zero) {                                                           \
                ACC br = b.re, bi = b.im, yr = y->re, yi = y->im;                    \
                zr = zr + (br * yr - bi * yi); /* + b*y */                           \
                zi = zi + (br * yi + bi * yr);                                       \
            }                                                                        \
            y->re = zr;                                                              \
            y->im = zi;                                                              \
        }                                                                            \
    }                                                                                \
}

O_CPLX_ONE(one_c, o_cfloat, float)
O_CPLX_ONE(one_z, o_cdouble, double)

#define O_CZERO(x) ((x).re == 0 && (x).im == 0)
#define O_CONE(x) ((x).re == 1 && (x).im == 0)

#define O_CPLX_API(SUF, CT)                                                             \
int oracle_gemm_batched_##SUF(char ta, char tb, int m, int n, int k, const CT *alpha,   \
                              const CT *A, int lda, long long lda2,                     \
                              const CT *B, int ldb, long long ldb2, const CT *beta,     \
                              CT *C, int ldc, long long ldc2, int batch)                \
{                                                                                       \
    int rc = validate(0, ta, tb, m, n, k, alpha, alpha && O_CZERO(*alpha), beta, A,     \
                      lda, lda2, B, ldb, ldb2, C, ldc, ldc2, batch, sizeof(CT), O_MAXDIM_CPLX);        \
    if (rc) return rc;                                                                  \
    CT a = *alpha, b = *beta;                                                           \
    if (m == 0 || n == 0 || batch == 0 || ((O_CZERO(a) || k == 0) && O_CONE(b)))        \
        return 0;                                                                       \
    if (k == 0) { a.re = 0; a.im = 0; }                                                 \
    for (int p = 0; p < batch; ++p)                                                     \
        one_##SUF(ta, tb, m, n, k, a, b, A + lda2 * p, lda, B + ldb2 * p, ldb,          \
                  C + ldc2 * p, ldc);                                                   \
    return 0;                                                                           \
}                                                                                       \
int oracle_gemm_batched_ptr_##SUF(char ta, char tb, int m, int n, int k,                \
                                  const CT *alpha, const CT *const *Aarray, int lda,    \
                                  const CT *const *Barray, int ldb, const CT *beta,     \
                                  CT *const *Carray, int ldc, int batch)                \
{                                                                                       \
    int rc = validate(1, ta, tb, m, n, k, alpha, alpha && O_CZERO(*alpha), beta,        \
                      Aarray, lda, 0, Barray, ldb, 0, Carray, ldc, 0, batch,            \
                      sizeof(CT), O_MAXDIM_CPLX);                                                      \
    if (rc) return rc;                                                                  \
    CT a = *alpha, b = *beta;                                                           \
    if (m == 0 || n == 0 || batch == 0 || ((O_CZERO(a) || k == 0) && O_CONE(b)))        \
        return 0;                                                                       \
    if (k == 0) { a.re = 0; a.im = 0; }                                                 \
    int rd = !O_CZERO(a);                                                               \
    for (int p = 0; p < batch; ++p)                                                     \
        one_##SUF(ta, tb, m, n, k, a, b, rd ? Aarray[p] : NULL, lda,                    \
                  rd ? Barray[p] : NULL, ldb, Carray[p], ldc);                          \
    return 0;                                                                           \
}

O_CPLX_API(c, o_cfloat)
O_CPLX_API(z, o_cdouble)

/* Sanity hooks for the Python wrapper. */
int oracle_abi_version(void) { return 1; }
