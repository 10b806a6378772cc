/*
 * txgemm.h -- C ABI of the B200-native batched small-matrix GEMM.
 *
 * Operation (§2 Eq. (1)), for p = 0 .. batch_count-1 independently:
 *
 *     C^p <- alpha * op(A^p) * op(B^p) + beta * C^p
 *
 *   op(X) = X, X^T or X^* selected by 'N'/'n', 'T'/'t', 'C'/'c' (PAPER.md:240-243,
 *   344-345); for the real types 'C' is the same as 'T'.  C^p is m x n, op(A^p) is
 *   m x k, op(B^p) is k x n; 0 <= m, n, k <= 64 for s and d,
 *   <= 32 for c and z (TX_MAX_DIM, TX_MAX_DIM_CPLX: about the FP32 / FP64 ridge
 *   point of each type, where the path stops being HBM-bound).  Sizes up to
 *   16 are the paper's regime and have ahead-of-time size-
 *   specialised kernels for square shapes; larger ones are the paper's "easily
 *   extended to larger sizes", served by runtime-
 *   specialised instances (reading R14).
 *   A is stored m x k when transa = 'N', else k x m; B is stored k x n when
 *   transb = 'N', else n x k (reading R8).  Storage is column-major.
 *
 * Types: s = float, d = double, c = tx_cfloat (layout of
 * cuComplex / float2 / torch.complex64), z = tx_cdouble (cuDoubleComplex /
 * double2 / torch.complex128).  Complex products use the 4-multiply/2-add
 * formula; the "3M" method is not used.
 *
 * Layouts.
 *  - Strided ("uniform", the paper's TGEMM_multi_uniform):
 *    entry (i, j) of matrix p of X is X[i + ldx*j + ldx2*p]; all leading
 *    dimensions are in ELEMENTS, not bytes.  ldx2 is 64-bit
 *    because p*ldx2 exceeds 2^31 at 10^7 16x16 pairs (reading R10).
 *    Inputs may use ld2 = 0 (one matrix broadcast to every p) and may overlap
 *    each other; C must satisfy ldc2 >= ldc*n (Fig. 1) and
 *    must not overlap A or B.
 *  - Pointer array ("nounif", cuBLAS-like): entry
 *    (i, j) of matrix p of X is Xarray[p][i + ldx*j].  Xarray is a DEVICE array
 *    of batch_count DEVICE pointers.  Output matrices must be pairwise disjoint
 *    and disjoint from the inputs (documented precondition, not checked: checking
 *    would need device reads).
 *
 * Memory and ownership.  The caller owns all memory; the library allocates no
 * device memory (the host-buffer entry creates two copy streams per device once,
 * and a few events per call).  A, B, C, the pointer arrays and their targets are device
 * memory of the CURRENT device.  alpha and beta are HOST pointers, read before
 * the call returns (the paper allows host or device; the
 * *_dev entries below take device-resident alpha/beta).
 *
 * Execution.  Asynchronous on `stream` (NULL = legacy default stream); returns
 * after enqueueing.  Reentrant and thread-safe.  Results are bitwise
 * deterministic for identical inputs and do not depend on the grid size.
 * beta == 0: C is write-only (never read, NaN in C does not propagate).
 * alpha == 0 or k == 0: A and B are never read; C <- beta*C.
 * Quick return, nothing enqueued: m == 0, n == 0, batch_count == 0, or
 * (alpha == 0 or k == 0) and beta == 1.
 *
 * Return value: 0 on success; -i when argument i (1-based position in the
 * call) is invalid -- nothing is enqueued and C is untouched; > 0 a cudaError_t
 * raised while launching.  Argument checks, in order (strided positions, the
 * pointer call's positions in brackets):
 *   transa -1, transb -2, m -3, n -4, k -5 (outside [0, TX_MAX_DIM] for s/d,
 *   [0, TX_MAX_DIM_CPLX] for c/z), alpha NULL -6,
 *   beta NULL -13 [-11], lda < max(1, rows of stored A) -8,
 *   ldb < max(1, rows of stored B) -11 [-10], ldc < max(1, m) -15 [-13];
 *   batch_count > 1 (strided only): lda2 < 0 -9, ldb2 < 0 -12, ldc2 < ldc*n -16;
 *   batch_count < 0 -17 [-14];
 *   A NULL or misaligned -7 / B -10 [-9] when alpha != 0, k > 0 and
 *   m*n*batch_count > 0; C NULL or misaligned -14 [-12] when m*n*batch_count > 0.
 *   "Misaligned" (reading R21): strided A, B, C must be aligned to the
 *   element size -- 4 (s), 8 (d), 8 (c), 16 (z) bytes, as float, double,
 *   cuComplex (float2) and cuDoubleComplex (double2) are -- because the kernels
 *   move whole elements; the pointer ARRAYS must be 8-byte aligned, and every
 *   pointer they hold must be aligned to the element size (documented
 *   precondition, not checked: it would need device reads);
 *   strided: C's address range overlapping A's or B's -14 (when A/B are read).
 */
#ifndef TXGEMM_H
#define TXGEMM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { float re, im; } tx_cfloat;
typedef struct { double re, im; } tx_cdouble;
/* Same handle as cudaStream_t / CUstream. */
typedef struct CUstream_st *tx_stream_t;

#define TX_VERSION 10100 /* 1.1.0 */
#define TX_MAX_DIM 64       /* s, d */
#define TX_MAX_DIM_CPLX 32  /* c, z */

/* ---- strided batch: TGEMM_multi_uniform. Args 1..18. ---- */
int tx_gemm_batched_s(char transa, char transb, int m, int n, int k,
                      const float *alpha, const float *A, int lda, long long lda2,
                      const float *B, int ldb, long long ldb2, const float *beta,
                      float *C, int ldc, long long ldc2, int batch_count, tx_stream_t stream);
int tx_gemm_batched_d(char transa, char transb, int m, int n, int k,
                      const double *alpha, const double *A, int lda, long long lda2,
                      const double *B, int ldb, long long ldb2, const double *beta,
                      double *C, int ldc, long long ldc2, int batch_count, tx_stream_t stream);
int tx_gemm_batched_c(char transa, char transb, int m, int n, int k,
                      const tx_cfloat *alpha, const tx_cfloat *A, int lda, long long lda2,
                      const tx_cfloat *B, int ldb, long long ldb2, const tx_cfloat *beta,
                      tx_cfloat *C, int ldc, long long ldc2, int batch_count, tx_stream_t stream);
int tx_gemm_batched_z(char transa, char transb, int m, int n, int k,
                      const tx_cdouble *alpha, const tx_cdouble *A, int lda, long long lda2,
                      const tx_cdouble *B, int ldb, long long ldb2, const tx_cdouble *beta,
                      tx_cdouble *C, int ldc, long long ldc2, int batch_count, tx_stream_t stream);

/* ---- pointer-array batch: TGEMM_multi_nounif. Args 1..15. ---- */
int tx_gemm_batched_ptr_s(char transa, char transb, int m, int n, int k, const float *alpha,
                          const float *const *Aarray, int lda, const float *const *Barray, int ldb,
                          const float *beta, float *const *Carray, int ldc, int batch_count,
                          tx_stream_t stream);
int tx_gemm_batched_ptr_d(char transa, char transb, int m, int n, int k, const double *alpha,
                          const double *const *Aarray, int lda, const double *const *Barray,
                          int ldb, const double *beta, double *const *Carray, int ldc,
                          int batch_count, tx_stream_t stream);
int tx_gemm_batched_ptr_c(char transa, char transb, int m, int n, int k, const tx_cfloat *alpha,
                          const tx_cfloat *const *Aarray, int lda,
                          const tx_cfloat *const *Barray, int ldb, const tx_cfloat *beta,
                          tx_cfloat *const *Carray, int ldc, int batch_count, tx_stream_t stream);
int tx_gemm_batched_ptr_z(char transa, char transb, int m, int n, int k,
                          const tx_cdouble *alpha, const tx_cdouble *const *Aarray, int lda,
                          const tx_cdouble *const *Barray, int ldb, const tx_cdouble *beta,
                          tx_cdouble *const *Carray, int ldc, int batch_count, tx_stream_t stream);

/* ---- host-buffer entry (end-to-end): same arguments and checks as the strided
 * call, except that hA, hB, hC are HOST pointers (pinned memory for overlap) and
 * dA, dB, dC (args 19, 20, 21) are caller-owned DEVICE staging buffers with the
 * same layouts (offsets and extents) as hA, hB, hC.  Enqueues on `stream`:
 * host->device copies of the A and B extents (and of C's extent when
 * beta != 0), the GEMM on the device copies, and the device->host copy of C's
 * extent back into hC.  The batch is processed in chunks of ~64 MB of traffic
 * (TX_HOSTIO_CHUNK_MB overrides; 4-512 MB measured, 64 best): host->device
 * copies run on an internal copy stream, device->host copies on another, the
 * GEMMs on `stream`, ordered by events, so both PCIe directions and the kernels
 * overlap; work already queued on `stream` is ordered before the first copy and
 * `stream` is ordered after the last one.  Returns as the strided call; a NULL
 * or misaligned staging buffer that would be used returns -19/-20/-21. ---- */
int tx_gemm_batched_hostio_s(char transa, char transb, int m, int n, int k,
                             const float *alpha, const float *hA, int lda, long long lda2,
                             const float *hB, int ldb, long long ldb2, const float *beta,
                             float *hC, int ldc, long long ldc2, int batch_count,
                             tx_stream_t stream, float *dA, float *dB, float *dC);
int tx_gemm_batched_hostio_d(char transa, char transb, int m, int n, int k,
                             const double *alpha, const double *hA, int lda, long long lda2,
                             const double *hB, int ldb, long long ldb2, const double *beta,
                             double *hC, int ldc, long long ldc2, int batch_count,
                             tx_stream_t stream, double *dA, double *dB, double *dC);
int tx_gemm_batched_hostio_c(char transa, char transb, int m, int n, int k,
                             const tx_cfloat *alpha, const tx_cfloat *hA, int lda,
                             long long lda2, const tx_cfloat *hB, int ldb, long long ldb2,
                             const tx_cfloat *beta, tx_cfloat *hC, int ldc, long long ldc2,
                             int batch_count, tx_stream_t stream, tx_cfloat *dA, tx_cfloat *dB,
                             tx_cfloat *dC);
int tx_gemm_batched_hostio_z(char transa, char transb, int m, int n, int k,
                             const tx_cdouble *alpha, const tx_cdouble *hA, int lda,
                             long long lda2, const tx_cdouble *hB, int ldb, long long ldb2,
                             const tx_cdouble *beta, tx_cdouble *hC, int ldc, long long ldc2,
                             int batch_count, tx_stream_t stream, tx_cdouble *dA,
                             tx_cdouble *dB, tx_cdouble *dC);

/* ---- device-resident alpha / beta (the paper's "host or device pointer",
 * PAPER.md:347, 354): identical to tx_gemm_batched_<t> / tx_gemm_batched_ptr_<t>
 * except that alpha and beta point to DEVICE memory and are read by the kernels
 * when they run (stream-ordered), so the call never synchronises.  The kernels
 * decide at run time: alpha == 0 -> C <- beta*C without reading A and B (nothing
 * when beta == 1); beta == 0 -> C is never read.  Because the values are not
 * known at the call, A and B must be valid whenever m*n*batch_count > 0 and
 * k > 0, and the overlap check of the strided call always applies.  Argument
 * positions and the other checks are those of the host-scalar calls. ---- */
int tx_gemm_batched_dev_s(char transa, char transb, int m, int n, int k, const float *alpha,
                          const float *A, int lda, long long lda2, const float *B, int ldb,
                          long long ldb2, const float *beta, float *C, int ldc, long long ldc2,
                          int batch_count, tx_stream_t stream);
int tx_gemm_batched_dev_d(char transa, char transb, int m, int n, int k, const double *alpha,
                          const double *A, int lda, long long lda2, const double *B, int ldb,
                          long long ldb2, const double *beta, double *C, int ldc, long long ldc2,
                          int batch_count, tx_stream_t stream);
int tx_gemm_batched_dev_c(char transa, char transb, int m, int n, int k, const tx_cfloat *alpha,
                          const tx_cfloat *A, int lda, long long lda2, const tx_cfloat *B, int ldb,
                          long long ldb2, const tx_cfloat *beta, tx_cfloat *C, int ldc,
                          long long ldc2, int batch_count, tx_stream_t stream);
int tx_gemm_batched_dev_z(char transa, char transb, int m, int n, int k, const tx_cdouble *alpha,
                          const tx_cdouble *A, int lda, long long lda2, const tx_cdouble *B,
                          int ldb, long long ldb2, const tx_cdouble *beta, tx_cdouble *C, int ldc,
                          long long ldc2, int batch_count, tx_stream_t stream);
int tx_gemm_batched_ptr_dev_s(char transa, char transb, int m, int n, int k, const float *alpha,
                              const float *const *Aarray, int lda, const float *const *Barray,
                              int ldb, const float *beta, float *const *Carray, int ldc,
                              int batch_count, tx_stream_t stream);
int tx_gemm_batched_ptr_dev_d(char transa, char transb, int m, int n, int k, const double *alpha,
                              const double *const *Aarray, int lda, const double *const *Barray,
                              int ldb, const double *beta, double *const *Carray, int ldc,
                              int batch_count, tx_stream_t stream);
int tx_gemm_batched_ptr_dev_c(char transa, char transb, int m, int n, int k,
                              const tx_cfloat *alpha, const tx_cfloat *const *Aarray, int lda,
                              const tx_cfloat *const *Barray, int ldb, const tx_cfloat *beta,
                              tx_cfloat *const *Carray, int ldc, int batch_count,
                              tx_stream_t stream);
int tx_gemm_batched_ptr_dev_z(char transa, char transb, int m, int n, int k,
                              const tx_cdouble *alpha, const tx_cdouble *const *Aarray, int lda,
                              const tx_cdouble *const *Barray, int ldb, const tx_cdouble *beta,
                              tx_cdouble *const *Carray, int ldc, int batch_count,
                              tx_stream_t stream);

/* ---- introspection and tuning (host only, no GPU work) ---- */
/* Human-readable text for a status code (static storage, never NULL). */
const char *tx_status_string(int status);
/* TX_VERSION of the built library. */
int tx_version(void);
/* Path the calling thread's most recent successful GEMM call took:
 * 0 none/quick return, 1 packed bulk-copy (TMA) kernel, 2 general gather kernel,
 * 3 pointer-array kernel, 4 scale-only kernel (alpha == 0 or k == 0),
 * 5 register-direct kernel (packed square n <= 2),
 * 6 tensor-core (tcgen05 split-TF32) kernel (packed s / c beyond 16);
 * +16 when a separate tail launch handled the last (< 16) pairs; +32 when the
 * kernel was a runtime-specialised (NVRTC, sm_100a) instance.  Also returns
 * the number of kernel launches of that call in *launches. */
int tx_last_path(int *launches);
/* Cap on CTAs per launch (0 = automatic: SMs x resident CTAs).  Results do not
 * depend on it; used for the grid-sweep experiment and determinism tests.
 * Process-wide; returns the previous value. */
int tx_set_max_ctas(int max_ctas);
/* Autotuning hook: force the bulk kernels' pipeline depth (2..8 stages) and
 * stage-size target (KB); 0 restores the per-instance table.  Process-wide;
 * returns the previous stage override.  Results do not depend on it. */
int tx_set_tuning(int stages, int stage_kb);
/* Runtime specialisation (NVRTC) of instances without an ahead-of-time kernel
 * (non-square sizes, pointer arrays, padded layouts): 1 enables (default, unless
 * TX_JIT=0 in the environment), 0 uses the generic-size AOT kernels.  Results are
 * bitwise identical either way.  Returns the previous setting. */
int tx_set_jit(int enable);
/* Tensor-core (tcgen05 split-TF32) kernel for packed s / c batches:
 * -1 = automatic (default: the sizes where the FP32 FMA pipe bounds the CUDA-core
 * kernels, or TX_TC=0/1 from the environment), 0 = never, 1 = wherever it applies
 * (m, n, k <= 64 for s, <= 32 for c).  Results differ from the CUDA-core kernels
 * only by rounding (same tolerance; bit-identical on integer-valued inputs).
 * Process-wide; returns the previous setting (-1 when automatic). */
int tx_set_tc(int mode);
/* Number of instances JIT-compiled by this process (cache misses), or -1 when
 * NVRTC is unavailable. */
int tx_jit_compiled(void);
/* Number of compiled kernel instances (AOT, size-specialised + generic). */
int tx_num_instances(void);

/* Layout classes for tx_prepare. */
#define TX_LAYOUT_PACKED 0  /* strided, minimal leading dimensions (ld = rows, ld2 = rows*cols) */
#define TX_LAYOUT_STRIDED 1 /* strided with padded ld / ld2 (the general gather kernel) */
#define TX_LAYOUT_PTR 2     /* pointer arrays of packed matrices */
/* Precompile: build (NVRTC) and load on the CURRENT device every runtime-
 * specialised instance that a call of type `type` ('s','d','c','z'), ops
 * transa/transb, sizes m, n, k, beta == 0 or not and layout class `layout`
 * would use, so that the first real call does no compilation (a first-use
 * compile otherwise takes seconds inside that call).  Launches nothing and
 * dereferences no memory.  Returns 0 (also when NVRTC is unavailable: the AOT
 * kernels need no preparation), -i for an invalid argument i (type -1,
 * transa -2, transb -3, m -4, n -5, k -6, layout -8), or > 0 a CUDA error. */
int tx_prepare(char type, char transa, char transb, int m, int n, int k, int beta_is_zero,
               int layout);

#ifdef __cplusplus
}
#endif

#endif /* TXGEMM_H */
