// tx_tc.cuh -- 5th-generation tensor-core (tcgen05, kind::tf32) path for the
// single-precision types (s, c) at the sizes beyond 16 where the FP32 FMA pipe,
// not HBM, bounds the CUDA-core kernels ("can be easily extended to larger
// sizes").
//
// Arithmetic: split-TF32 ("3xTF32").  Each fp32 operand x is split into
//   hi = rna_tf32(x),  lo = x - hi (exact in fp32; the tensor core truncates it to tf32)
// and  C^p = alpha * (A_hi B_lo + A_lo B_hi + A_hi B_hi) + beta * C^p,
// the three products accumulated in fp32 in TMEM by tcgen05.mma (the dropped
// A_lo B_lo term and the truncation of lo are O(2^-21) relative to |a||b|).
// Integer-valued inputs (|x| < 2^11) have lo = 0 and exact products, so the
// result is exact whenever the true sums are (bit-exact tests).
//
// Complex (c) in real form, rows interleaved (re, im):
//   X = [Ar_0; Ai_0; Ar_1; Ai_1; ...],  Y = [-Ai_0; Ar_0; -Ai_1; Ar_1; ...]   (2m x k)
//   D = X Br + Y Bi  ->  D[2i] = Re C_i.,  D[2i+1] = Im C_i.                 (2m x n)
// with Ai -> -Ai for op(A) = 'C' and Bi -> -Bi for op(B) = 'C'.
//
// MMA shape: M = 64 (the A-side rows: m real, 2m complex; <= 64), N = roundup(n, 8),
// K = 8 per instruction; operands in shared memory (K-major, 128-byte swizzle).
// With both operands read from shared memory an MMA costs (64 + N) * 32 B of
// shared-memory bandwidth, which M = 128 would double on the A side for rows the
// matrices do not have.  Accumulator row r sits in TMEM lane 32 * (r / 16) + r % 16
// (tools/tc_probe.py), so the 4 epilogue warps each own 16 rows.
//
// Per CTA (persistent, 448 threads, warp-specialised, mbarrier hand-offs only):
//   producer (1 thread)  packed tiles of P pairs -> S-stage ring (1-D bulk copies)
//   transform (8 warps)  each pair's op(A), op(B) -> hi/lo canonical layouts in one of
//                        NU operand units (one unit per K-block of 32)
//   MMA (1 thread)       3 (real) / 6 (complex) MMAs per K-step of 8 into one of 4
//                        TMEM accumulators, tcgen05.commit -> mbarriers
//   epilogue (4 warps)   tcgen05.ld -> alpha / beta (C from the stage) -> st.global
#pragma once
#include "tx_kernels.cuh"

namespace tx {

#ifdef TC_TRACE
__device__ unsigned long long tc_trace[8][256];  // [event][index]: clock64, CTA 0
#define TC_T(ev, idx)                                                     \
    do {                                                                   \
        if (blockIdx.x == 0 && (idx) < 256) tc_trace[ev][idx] = clock64(); \
    } while (0)
#else
#define TC_T(ev, idx) \
    do {              \
    } while (0)
#endif

template <class T> struct TcOk { static constexpr bool value = false; };
template <> struct TcOk<float> { static constexpr bool value = true; };
template <> struct TcOk<float2> { static constexpr bool value = true; };

constexpr int TC_TG = 256;             // transform threads (8 warps)
constexpr int TC_EW = 8;               // epilogue warps (2 per TMEM lane quadrant)
constexpr int TC_W_TR0 = TC_EW;        // first transform warp
constexpr int TC_W_PROD = TC_W_TR0 + TC_TG / 32, TC_W_MMA = TC_W_PROD + 1, TC_W_CPROD = TC_W_PROD + 2;
constexpr int TC_NT = 32 * (TC_W_CPROD + 1);  // 19 warps
constexpr int TC_CSMAX = 8;            // C stages (ring)
constexpr int TC_NUMAX = 4;            // operand units (ring)
constexpr int TC_NACC = 4;             // TMEM accumulators (ring)
constexpr int TC_ACC_COLS = 64;        // columns per accumulator (N <= 64)
constexpr int TC_TMEM_COLS = 256;
constexpr int TC_M = 64;
#ifndef TC_SUSPEND_NS
#define TC_SUSPEND_NS 1000000
#endif

// Shared-memory layout of one operand unit (one K-block of <= 32 elements).
//   real:    [A_hi | A_lo | B_hi | B_lo]            A: 64 rows, B: N rows, 128 B each
//   complex: [X_hi | Y_hi | X_lo | Y_lo | Br_hi | Bi_hi | Br_lo | Bi_lo]
// bytes of a stage window for `bytes` operand bytes starting at any 4-byte offset
__host__ __device__ inline int tc_win(int bytes) { return (bytes + 15 + 15) & ~15; }

struct TcGeom {
    int N;       // MMA N = roundup(n, 8)
    int KB;      // K-blocks of 32 elements per pair (complex: k <= 32 -> 1)
    int K8;      // roundup(k, 8)
    int abytes;  // one A-side array (64 rows x 128 B)
    int bbytes;  // one B-side array (N rows x 128 B)
    int unit;    // one operand unit
};

__host__ __device__ inline TcGeom tc_geom(bool cplx, int m, int n, int k)
{
    (void)m;
    TcGeom g;
    g.N = cplx ? (2 * n + 7) & ~7 : (n + 7) & ~7;
    g.K8 = (k + 7) & ~7;
    g.KB = (k + 31) / 32;
    g.abytes = TC_M * 128;
    g.bbytes = g.N * 128;
    g.unit = 2 * g.abytes + 2 * g.bbytes;
    return g;
}

// byte offset of 16-byte chunk c of row r in a K-major SW128 array: 8-row groups
// 1024 B apart, chunk c of row r stored at chunk position c ^ (r mod 8).
__device__ __forceinline__ uint32_t tc_off(int r, int c)
{
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((c ^ r) & 7) << 4));
}

// hi = x rounded to tf32 (nearest, ties away from zero: the mantissa bits below the
// tf32 ones are rounded by adding half an ulp and masking) -- two integer operations
// instead of cvt.rna.tf32.f32's four (its extra two only special-case Inf/NaN, which
// stay Inf/NaN here too, a NaN whose payload sits below bit 13 becoming Inf with lo = NaN).
// lo = x - hi is exact in fp32 and is left to the tensor core's own truncation to tf32
// (probe: RZ), |x - hi - trunc(x - hi)| < 2^-21 |x|.
__device__ __forceinline__ float tf32_hi(float x)
{
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// hi / lo parts of 4 values -> two 16-byte shared stores
__device__ __forceinline__ void tc_put4(unsigned char *hi, unsigned char *lo, uint32_t off, float v0,
                                        float v1, float v2, float v3)
{
    const float h0 = tf32_hi(v0), h1 = tf32_hi(v1), h2 = tf32_hi(v2), h3 = tf32_hi(v3);
    *reinterpret_cast<float4 *>(hi + off) = make_float4(h0, h1, h2, h3);
    *reinterpret_cast<float4 *>(lo + off) = make_float4(v0 - h0, v1 - h1, v2 - h2, v3 - h3);
}

// the same for a complex operand row pair: X gets (v), Y gets (sy * v), sy = +-1
__device__ __forceinline__ void tc_put4xy(unsigned char *xhi, unsigned char *xlo, uint32_t xo,
                                          unsigned char *yhi, unsigned char *ylo, uint32_t yo,
                                          float sy, const float (&v)[4])
{
    float h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        h[q] = tf32_hi(v[q]);
        l[q] = v[q] - h[q];
    }
    *reinterpret_cast<float4 *>(xhi + xo) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4 *>(xlo + xo) = make_float4(l[0], l[1], l[2], l[3]);
    *reinterpret_cast<float4 *>(yhi + yo) = make_float4(sy * h[0], sy * h[1], sy * h[2], sy * h[3]);
    *reinterpret_cast<float4 *>(ylo + yo) = make_float4(sy * l[0], sy * l[1], sy * l[2], sy * l[3]);
}

// Shared-memory matrix descriptor (tcgen05): K-major, 128-byte swizzle, SBO = 1024.
// The start address is the low 14 bits (16-byte units), so the descriptor of
// addr + off is tc_desc(addr) + off / 16 for the offsets used here.
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: kind::tf32, fp32 accumulator, both operands K-major.
__device__ __forceinline__ uint32_t tc_idesc(int M, int N)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// mbarrier wait with a suspend-time hint: a waiting thread sleeps until the phase
// completes (or the hint expires) instead of spinning on the issue slots the
// transform and epilogue warps need.
__device__ __forceinline__ void tc_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra TC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(TC_SUSPEND_NS)
        : "memory");
}

// (mbar_arrive: tx_common.cuh)
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 accumulator columns of this warp's 32 TMEM lanes (issue; tc_ld_wait before use)
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
        " [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tc_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- transform
// Work items are 16-byte chunks (4 consecutive K elements) of one operand row.
// Thread decomposition by shifts (no divisions): when the stored matrix is
// contiguous along the operand rows, consecutive threads take consecutive rows
// (conflict-free reads, and 8 consecutive rows hit 8 distinct swizzled chunk
// positions); when it is contiguous along K, 8 consecutive threads take the 8
// chunks of one row.
__device__ __forceinline__ int tc_log2ceil(int x)
{
    int s = 0;
    while ((1 << s) < x) ++s;
    return s;
}

// Real: op(A) (m x k) and op(B) (k x n) of one pair, K-block kb.
template <int OPA, int OPB>
__device__ __forceinline__ void tc_transform_real(const float *__restrict__ sA,
                                                  const float *__restrict__ sB, unsigned char *u,
                                                  const TcGeom &g, int m, int n, int k, int kb,
                                                  int tid, bool veca, bool vecb, int shm, int shn)
{
    const int k0 = kb * 32;
    const int KC = min(32, g.K8 - k0) >> 2;  // 16-byte chunks per row in this block
    unsigned char *ahi = u, *alo = u + g.abytes, *bhi = u + 2 * g.abytes, *blo = bhi + g.bbytes;
    // A: element (i, l) = OPA == N ? sA[i + m*l] : sA[l + k*i]
    if (OPA == OP_N) {
        const int sh = shm;
        const int i = tid & ((1 << sh) - 1);
        if (i < m)
            for (int c = tid >> sh; c < KC; c += TC_TG >> sh) {
                const int l = k0 + 4 * c;
                float v[4];
                if (l + 3 < k) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = sA[i + m * (l + e)];
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = (l + e < k) ? sA[i + m * (l + e)] : 0.f;
                }
                tc_put4(ahi, alo, tc_off(i, c), v[0], v[1], v[2], v[3]);
            }
    } else {
        const int c = tid & 7;
        if (c < KC)
            for (int i = tid >> 3; i < m; i += TC_TG >> 3) {
                const int l = k0 + 4 * c;
                float v[4];
                if (veca && l + 3 < k) {
                    const float4 t = *reinterpret_cast<const float4 *>(sA + l + k * i);
                    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = (l + e < k) ? sA[(l + e) + k * i] : 0.f;
                }
                tc_put4(ahi, alo, tc_off(i, c), v[0], v[1], v[2], v[3]);
            }
    }
    // B: operand row j = column j of op(B); element (l, j) = OPB == N ? sB[l + k*j] : sB[j + n*l]
    if (OPB == OP_N) {
        const int c = tid & 7;
        if (c < KC)
            for (int j = tid >> 3; j < n; j += TC_TG >> 3) {
                const int l = k0 + 4 * c;
                float v[4];
                if (vecb && l + 3 < k) {
                    const float4 t = *reinterpret_cast<const float4 *>(sB + l + k * j);
                    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = (l + e < k) ? sB[(l + e) + k * j] : 0.f;
                }
                tc_put4(bhi, blo, tc_off(j, c), v[0], v[1], v[2], v[3]);
            }
    } else {
        const int sh = shn;
        const int j = tid & ((1 << sh) - 1);
        if (j < n)
            for (int c = tid >> sh; c < KC; c += TC_TG >> sh) {
                const int l = k0 + 4 * c;
                float v[4];
                if (l + 3 < k) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = sB[j + n * (l + e)];
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = (l + e < k) ? sB[j + n * (l + e)] : 0.f;
                }
                tc_put4(bhi, blo, tc_off(j, c), v[0], v[1], v[2], v[3]);
            }
    }
}

// Complex: X (rows 2i + e: (ar, sa*ai) of op(A) row i) and B' (rows j: br of op(B)
// column j; rows n + j: sb*bi), k <= 32 (one K-block).
template <int OPA, int OPB>
__device__ __forceinline__ void tc_transform_cplx(const float2 *__restrict__ sA,
                                                  const float2 *__restrict__ sB, unsigned char *u,
                                                  const TcGeom &g, int m, int n, int k, int tid,
                                                  bool veca, bool vecb, int shm, int shn)
{
    const int KC = g.K8 >> 2;
    unsigned char *xhi = u, *xlo = u + g.abytes, *bhi = u + 2 * g.abytes, *blo = bhi + g.bbytes;
    constexpr float sa = OPA == OP_C ? -1.f : 1.f, sb = OPB == OP_C ? -1.f : 1.f;
    auto put_a = [&](int i, int e, int c, const float2 (&a)[4]) {
        if (e)
            tc_put4(xhi, xlo, tc_off(2 * i + 1, c), sa * a[0].y, sa * a[1].y, sa * a[2].y, sa * a[3].y);
        else
            tc_put4(xhi, xlo, tc_off(2 * i, c), a[0].x, a[1].x, a[2].x, a[3].x);
    };
    if (OPA == OP_N) {
        const int sh = shm + 1;
        const int e = tid & 1, i = (tid & ((1 << sh) - 1)) >> 1;
        if (i < m)
            for (int c = tid >> sh; c < KC; c += TC_TG >> sh) {
                const int l = 4 * c;
                float2 a[4];
                if (l + 3 < k) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) a[q] = sA[i + m * (l + q)];
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        a[q] = (l + q < k) ? sA[i + m * (l + q)] : make_float2(0.f, 0.f);
                }
                put_a(i, e, c, a);
            }
    } else {
        const int c = tid & 7, e = (tid >> 3) & 1;
        if (c < KC)
            for (int i = tid >> 4; i < m; i += TC_TG >> 4) {
                const int l = 4 * c;
                float2 a[4];
                if (veca && l + 3 < k) {
                    const float4 *p = reinterpret_cast<const float4 *>(sA + l + k * i);
                    const float4 t0 = p[0], t1 = p[1];
                    a[0] = make_float2(t0.x, t0.y); a[1] = make_float2(t0.z, t0.w);
                    a[2] = make_float2(t1.x, t1.y); a[3] = make_float2(t1.z, t1.w);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        a[q] = (l + q < k) ? sA[(l + q) + k * i] : make_float2(0.f, 0.f);
                }
                put_a(i, e, c, a);
            }
    }
    auto put_b = [&](int j, int c, const float2 (&b)[4]) {
        tc_put4(bhi, blo, tc_off(j, c), b[0].x, b[1].x, b[2].x, b[3].x);
        tc_put4(bhi, blo, tc_off(n + j, c), sb * b[0].y, sb * b[1].y, sb * b[2].y, sb * b[3].y);
    };
    if (OPB == OP_N) {
        const int c = tid & 7;
        if (c < KC)
            for (int j = tid >> 3; j < n; j += TC_TG >> 3) {
                const int l = 4 * c;
                float2 b[4];
                if (vecb && l + 3 < k) {
                    const float4 *p = reinterpret_cast<const float4 *>(sB + l + k * j);
                    const float4 t0 = p[0], t1 = p[1];
                    b[0] = make_float2(t0.x, t0.y); b[1] = make_float2(t0.z, t0.w);
                    b[2] = make_float2(t1.x, t1.y); b[3] = make_float2(t1.z, t1.w);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        b[q] = (l + q < k) ? sB[(l + q) + k * j] : make_float2(0.f, 0.f);
                }
                put_b(j, c, b);
            }
    } else {
        const int sh = shn;
        const int j = tid & ((1 << sh) - 1);
        if (j < n)
            for (int c = tid >> sh; c < KC; c += TC_TG >> sh) {
                const int l = 4 * c;
                float2 b[4];
                if (l + 3 < k) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) b[q] = sB[j + n * (l + q)];
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        b[q] = (l + q < k) ? sB[j + n * (l + q)] : make_float2(0.f, 0.f);
                }
                put_b(j, c, b);
            }
    }
}

// MMAs of one operand unit into the accumulator at `tmem` (one thread).
template <bool CPLX>
__device__ __forceinline__ void tc_issue(uint32_t ubase, const TcGeom &g, int kb, uint32_t tmem)
{
    const uint32_t id = tc_idesc(TC_M, g.N);
    const int ksteps = min(32, g.K8 - kb * 32) >> 3;
    const uint64_t d0 = tc_desc(ubase);
    const uint32_t A = (uint32_t)g.abytes >> 4, B = (uint32_t)g.bbytes >> 4;  // 16-byte units
    for (int s = 0; s < ksteps; ++s) {
        const uint64_t d = d0 + (uint64_t)(s * 2);  // 8 tf32 = 32 bytes along K in the atom
        const uint32_t first = (kb == 0 && s == 0) ? 0u : 1u;
        (void)CPLX;  // complex: the same three products, X against B' = [Br | Bi]
        const uint64_t ahi = d, alo = d + A, bhi = d + 2 * A, blo = bhi + B;
        tc_mma(tmem, ahi, blo, id, first);
        tc_mma(tmem, alo, bhi, id, 1u);
        tc_mma(tmem, ahi, bhi, id, 1u);
    }
}

// Epilogue of one pair by epilogue warp (q, h): accumulator rows 16q .. 16q+15 (TMEM
// lanes 32q .. 32q+15; q = warp % 4), column chunks h, h + 2, ... of 16 -> alpha/beta ->
// C (column-major, ld = m).
template <class T, bool B0>
__device__ __forceinline__ void tc_epilogue(uint32_t tacc, const T *__restrict__ sC,
                                            T *__restrict__ gC, int m, int n, int q, int h, int lane,
                                            T alpha, T beta)
{
    constexpr bool CPLX = same_t<T, float2>::value;
    const int rows = CPLX ? 2 * m : m;
    if (q * 16 >= rows) return;  // warp-uniform
    const int r = q * 16 + (lane & 15);
    const bool live = lane < 16 && r < rows;
    const uint32_t lane_addr = tacc + ((uint32_t)(q * 32) << 16);
    for (int c0 = 16 * h; c0 < n; c0 += 16 * (TC_EW / 4)) {  // column chunks dealt to the
        const int cnt = min(16, n - c0);                       // warps of this quadrant
        uint32_t v[16];
        tc_ld16(lane_addr + c0, v);
        if constexpr (!CPLX) {
            const float *sc = B0 ? nullptr : sC + r + m * c0;
            float *gc = gC + r + (long long)m * c0;
            float cin[16];
            if (!B0 && live) {
                if (cnt == 16) {
#pragma unroll
                    for (int t = 0; t < 16; ++t) cin[t] = sc[t * m];
                } else {
#pragma unroll
                    for (int t = 0; t < 16; ++t) cin[t] = t < cnt ? sc[t * m] : 0.f;
                }
            }
            tc_ld_wait();
            if (live) {
#pragma unroll
                for (int t = 0; t < 16; ++t)
                    if (t < cnt) {
                        const float x = __uint_as_float(v[t]);
                        gc[t * m] = B0 ? ax(alpha, x) : axpby(alpha, x, beta, cin[t]);
                    }
            }
        } else {
            // lane pair (2i, 2i+1): the even lane holds ArBr, ArBi of row i, the odd lane
            // AiBr, AiBi; the even lane finishes the even columns, the odd lane the odd ones
            uint32_t w[16];
            tc_ld16(lane_addr + n + c0, w);  // the Bi half of the accumulator
            const int i = r >> 1, e = r & 1;
            const float2 *sc = B0 ? nullptr : sC + i + m * (c0 + e);
            float2 *gc = gC + i + (long long)m * (c0 + e);
            float2 cin[8];
            if (!B0 && live) {
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    cin[t] = 2 * t + e < cnt ? sc[2 * t * m] : make_float2(0.f, 0.f);
            }
            tc_ld_wait();
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float xr0 = __uint_as_float(v[2 * t]), xr1 = __uint_as_float(v[2 * t + 1]);
                const float xi0 = __uint_as_float(w[2 * t]), xi1 = __uint_as_float(w[2 * t + 1]);
                // the partner's values of this lane's column: even lanes send column 2t+1,
                // odd lanes column 2t
                const float sr = e ? xr0 : xr1, si = e ? xi0 : xi1;
                const float pr = __shfl_xor_sync(0xffffffffu, sr, 1);
                const float pi = __shfl_xor_sync(0xffffffffu, si, 1);
                if (live && 2 * t + e < cnt) {
                    const float arbr = e ? pr : xr0, arbi = e ? pi : xi0;
                    const float aibr = e ? xr1 : pr, aibi = e ? xi1 : pi;
                    const float2 x = make_float2(arbr - aibi, arbi + aibr);
                    gc[2 * t * m] = B0 ? ax(alpha, x) : axpby(alpha, x, beta, cin[t]);
                }
            }
        }
    }
}

// Warp roles: warps 0-7 epilogue (warp w reads TMEM lane quadrant w % 4, column chunks
// w / 4, w / 4 + 2, ...), warps 8-15 transform, warp 16 lane 0 A/B producer, warp 17
// lane 0 MMA issuer, warp 18 lane 0 C producer (beta != 0).  Two rings, so an A/B stage is recycled as soon as it is
// transformed (its lifetime no longer includes the MMAs and the epilogue):
//   full[s] / sfree[s]   A/B stage s landed / transformed (8 arrivals)
//   cfull[c] / cfree[c]  C stage c landed / read by the epilogue (8 arrivals)
//   uready[b] / ufree[b] operand unit b written (8 arrivals) / its MMAs completed (commit)
//   aready[a] / afree[a] accumulator a finished (commit) / read out (8 arrivals)
// p.S packs the A/B stages (bits 0-7), the operand units (8-15) and the C stages (16-23).
template <class T, int OPA, int OPB, bool B0>
__global__ void __launch_bounds__(TC_NT, 1) tc_kernel(const __grid_constant__ Params<T> p)
{
    static_assert(TcOk<T>::value, "tc_kernel: float / float2");
    constexpr bool CPLX = same_t<T, float2>::value;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int m = p.m, n = p.n, k = p.k;
    const TcGeom g = tc_geom(CPLX, m, n, k);
    const int KB = CPLX ? 1 : g.KB;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int P = p.P, S = p.S & 0xFF, NU = (p.S >> 8) & 0xFF, CS = (p.S >> 16) & 0xFF;
    const int ES = (int)sizeof(T);
    // A/B stage: [A window | B window]; C stage: [C window].  A window is the 16-byte-
    // aligned byte range covering the tile's contiguous operand bytes (any element-aligned
    // base: the operand starts (addr & 15) bytes into its window).
    const int offB = tc_win(P * SA * ES);
    const int stage_bytes = (offB + tc_win(P * SB * ES) + 1023) & ~1023;
    const int cstage_bytes = (tc_win(P * SC * ES) + 127) & ~127;
    const uintptr_t gA = reinterpret_cast<uintptr_t>(p.A), gB = reinterpret_cast<uintptr_t>(p.B),
                    gCin = reinterpret_cast<uintptr_t>(p.C);
    // 1024-byte aligned base, derived from the shared array (keeps the shared state space)
    unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char *ubuf = base + S * stage_bytes;   // NU operand units (1024-aligned)
    unsigned char *cbuf = ubuf + NU * g.unit;       // CS C stages
    uint64_t *bars = reinterpret_cast<uint64_t *>(cbuf + CS * cstage_bytes);
    uint64_t *full = bars, *sfree = bars + S, *uready = bars + 2 * S, *ufree = uready + TC_NUMAX,
             *aready = ufree + TC_NUMAX, *afree = aready + TC_NACC, *cfull = afree + TC_NACC,
             *cfree = cfull + TC_CSMAX;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(cfree + TC_CSMAX);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&sfree[s], TC_TG / 32);
        }
        for (int c = 0; c < TC_CSMAX; ++c) {
            mbar_init(&cfull[c], 1);
            mbar_init(&cfree[c], TC_EW);
        }
        for (int b = 0; b < TC_NUMAX; ++b) {
            mbar_init(&uready[b], TC_TG / 32);
            mbar_init(&ufree[b], 1);
        }
        for (int a = 0; a < TC_NACC; ++a) {
            mbar_init(&aready[a], 1);
            mbar_init(&afree[a], TC_EW);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(TC_TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_wait();
    grid_dep_launch();
    auto tile_pairs = [&](int i) {
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        return (int)min((long long)P, p.batch - pair0);
    };
    // bulk copy of the 16-byte-aligned window covering [addr, addr + bytes)
    auto window = [&](unsigned char *dst, uintptr_t addr, int bytes, uint64_t *bar, uint64_t pol) {
        const uint32_t wb = (uint32_t)(((addr & 15) + (uintptr_t)bytes + 15) & ~(uintptr_t)15);
        bulk_g2s(dst, reinterpret_cast<const void *>(addr & ~(uintptr_t)15), wb, bar, pol);
        return wb;
    };

    // ring cursors: slot index and phase parity, advanced without divisions; a wait for
    // a free slot uses parity phase ^ 1, which a fresh mbarrier reports complete
    struct Cur {
        int i = 0, ph = 0;
        __device__ __forceinline__ void next(int n)
        {
            if (++i == n) {
                i = 0;
                ph ^= 1;
            }
        }
    };
    if (warp == TC_W_PROD) {  // ----------------------------------------- A/B producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            Cur st_;
            for (int i = 0; i < my_tiles; ++i, st_.next(S)) {
                tc_wait(&sfree[st_.i], st_.ph ^ 1);
                TC_T(0, i);
                const long long pair0 = (blockIdx.x + (long long)i * G) * P;
                const int np = tile_pairs(i);
                unsigned char *st = base + st_.i * stage_bytes;
                const uintptr_t a0 = gA + pair0 * SA * ES, b0 = gB + pair0 * SB * ES;
                const uint32_t wa = (uint32_t)(((a0 & 15) + np * SA * ES + 15) & ~15ull),
                               wb = (uint32_t)(((b0 & 15) + np * SB * ES + 15) & ~15ull);
                mbar_arrive_expect_tx(&full[st_.i], wa + wb);
                window(st, a0, np * SA * ES, &full[st_.i], pol);
                window(st + offB, b0, np * SB * ES, &full[st_.i], pol);
            }
        }
    } else if (warp == TC_W_CPROD) {  // ----------------------------------- C producer
        if (!B0 && lane == 0) {
            const uint64_t pol = policy_evict_first();
            Cur cs_;
            for (int i = 0; i < my_tiles; ++i, cs_.next(CS)) {
                tc_wait(&cfree[cs_.i], cs_.ph ^ 1);
                const long long pair0 = (blockIdx.x + (long long)i * G) * P;
                const int np = tile_pairs(i);
                const uintptr_t c0 = gCin + pair0 * SC * ES;
                const uint32_t wc = (uint32_t)(((c0 & 15) + np * SC * ES + 15) & ~15ull);
                mbar_arrive_expect_tx(&cfull[cs_.i], wc);
                window(cbuf + cs_.i * cstage_bytes, c0, np * SC * ES, &cfull[cs_.i], pol);
            }
        }
    } else if (warp == TC_W_MMA) {  // --------------------------------------- MMA issuer
        if (lane == 0) {
            Cur un, ac;
            int u = 0;
            for (int i = 0; i < my_tiles; ++i) {
                const int np = tile_pairs(i);
                for (int q = 0; q < np; ++q, ac.next(TC_NACC)) {
                    const uint32_t acc = tmem + (uint32_t)(ac.i * TC_ACC_COLS);
                    tc_wait(&afree[ac.i], ac.ph ^ 1);
                    for (int kb = 0; kb < KB; ++kb, ++u, un.next(NU)) {
                        tc_wait(&uready[un.i], un.ph);
                        TC_T(3, u);
                        tc_fence_after();
#ifndef TC_EXP_NOMMA
                        tc_issue<CPLX>(smem_u32(ubuf + un.i * g.unit), g, kb, acc);
#endif
                        tc_commit(&ufree[un.i]);
                        TC_T(4, u);
                    }
                    tc_commit(&aready[ac.i]);
                }
            }
        }
    } else if (warp >= TC_W_TR0 && warp < TC_W_TR0 + TC_TG / 32) {  // ------- transform
        const int tg = tid - TC_W_TR0 * 32;
        const int shm = tc_log2ceil(m), shn = tc_log2ceil(n);
        Cur st_, un;
        int u = 0;
        for (int i = 0; i < my_tiles; ++i, st_.next(S)) {
            const int np = tile_pairs(i);
            const unsigned char *st = base + st_.i * stage_bytes;
            tc_wait(&full[st_.i], st_.ph);
            const long long pair0 = (blockIdx.x + (long long)i * G) * P;
            const int oa = (int)((gA + pair0 * SA * ES) & 15), ob = (int)((gB + pair0 * SB * ES) & 15);
            // 16-byte vector reads of a row need a 16-byte aligned window start
            const bool veca = oa == 0 && (CPLX ? (k & 1) == 0 : (k & 3) == 0);
            const bool vecb = ob == 0 && (CPLX ? (k & 1) == 0 : (k & 3) == 0);
            for (int q = 0; q < np; ++q) {
                const T *sA = reinterpret_cast<const T *>(st + oa) + q * SA;
                const T *sB = reinterpret_cast<const T *>(st + offB + ob) + q * SB;
                for (int kb = 0; kb < KB; ++kb, ++u, un.next(NU)) {
                    tc_wait(&ufree[un.i], un.ph ^ 1);
                    if (tg == 0) TC_T(1, u);
                    unsigned char *ub = ubuf + un.i * g.unit;
#ifndef TC_EXP_NOTRANSFORM  // (measurement builds of tools/tc_trace.cu only)
                    if constexpr (CPLX)
                        tc_transform_cplx<OPA, OPB>(sA, sB, ub, g, m, n, k, tg, veca, vecb, shm, shn);
                    else
                        tc_transform_real<OPA, OPB>(sA, sB, ub, g, m, n, k, kb, tg, veca, vecb, shm,
                                                    shn);
#endif
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&uready[un.i]);
                    if (tg == 0) TC_T(2, u);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sfree[st_.i]);  // the stage's A and B are in operand units
        }
    } else if (warp < TC_EW) {  // ------------------------------------------- epilogue
        const T alpha = p.alpha, beta = p.beta;
        Cur ac, cs_;
        int pp = 0;
        for (int i = 0; i < my_tiles; ++i) {
            const int np = tile_pairs(i);
            const long long pair0 = (blockIdx.x + (long long)i * G) * P;
            const T *sCt = nullptr;
            if (!B0) {
                tc_wait(&cfull[cs_.i], cs_.ph);
                const int oc = (int)((gCin + pair0 * SC * ES) & 15);
                sCt = reinterpret_cast<const T *>(cbuf + cs_.i * cstage_bytes + oc);
            }
            for (int q = 0; q < np; ++q, ++pp, ac.next(TC_NACC)) {
                tc_wait(&aready[ac.i], ac.ph);
                if (warp == 0 && lane == 0) TC_T(5, pp);
                tc_fence_after();
#ifndef TC_EXP_NOEPI
                tc_epilogue<T, B0>(tmem + (uint32_t)(ac.i * TC_ACC_COLS), B0 ? nullptr : sCt + q * SC,
                                   p.C + (pair0 + q) * SC, m, n, warp & 3, warp >> 2, lane, alpha,
                                   beta);
#endif
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afree[ac.i]);
                if (warp == 0 && lane == 0) TC_T(6, pp);
            }
            if (!B0) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&cfree[cs_.i]);
                cs_.next(CS);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(TC_TMEM_COLS)
                     : "memory");
    }
}

// Host plan of the tensor-core kernel: P pairs per tile, S A/B stages, NU operand
// units and CS C stages (beta != 0) within 227 KB.  NU = 3 when it fits (the
// transform runs up to two units ahead of the tensor core); A/B stages until S - 1 of
// them in flight cover >= 48 KB (the HBM latency-bandwidth product of one SM); C
// stages S + 2 (a tile's C is read two to three tiles after its A/B).
struct TcPlan {
    int P, S, NU, CS, smem, ntiles;
};

inline int tc_smem_bytes(bool cplx, int es, int m, int n, int k, bool b0, int P, int S, int NU,
                         int CS)
{
    const TcGeom g = tc_geom(cplx, m, n, k);
    const int stage = (tc_win(P * m * k * es) + tc_win(P * k * n * es) + 1023) & ~1023;
    const int cstage = b0 ? 0 : ((tc_win(P * m * n * es) + 127) & ~127);
    return 1024 + S * stage + NU * g.unit + CS * cstage +
           (2 * S + 2 * TC_NUMAX + 2 * TC_NACC + 2 * TC_CSMAX) * 8 + 16;
}

inline bool tc_plan(bool cplx, int es, int m, int n, int k, bool b0, int batch, TcPlan &pl)
{
    const int ab_bytes = (m * k + k * n) * es;
    // prefer (in order): A/B bytes in flight >= 48 KB with 3 operand units, the same with
    // 2 units, then the most A/B stages that fit
    for (int pass = 0; pass < 3; ++pass) {
        const int NU = pass == 0 ? 3 : 2;
        for (int P = 1; P <= 64; ++P) {
            int S = 0, CS = 0;
            for (int s = 6; s >= 2 && !S; --s) {
                const int cs = b0 ? 0 : std::min(TC_CSMAX, s + 2);
                for (int c = cs; c >= (b0 ? 0 : 2) && !S; --c)
                    if (tc_smem_bytes(cplx, es, m, n, k, b0, P, s, NU, c) <= SMEM_MAX_BYTES) {
                        S = s;
                        CS = c;
                    }
            }
            if (S == 0) break;
            const bool flight = (long long)(S - 1) * P * ab_bytes >= 48 * 1024;
            if (flight || pass == 2) {
                const int sms = num_sms();  // keep every SM busy for small batches
                int PP = P;
                while (PP > 1 && (long long)(batch + PP - 1) / PP < sms) --PP;
                pl.P = PP;
                pl.S = S;
                pl.NU = NU;
                pl.CS = CS;
                pl.smem = tc_smem_bytes(cplx, es, m, n, k, b0, pl.P, S, NU, CS);
                pl.ntiles = (int)(((long long)batch + pl.P - 1) / pl.P);
                return true;
            }
        }
    }
    return false;
}

// Launch (packed layout: ld = rows, ld2 = rows * cols; element-aligned operands; any batch).
template <class T, int OPA, int OPB, bool B0>
cudaError_t launch_tc(const void *vp, cudaStream_t st)
{
    Params<T> p = *static_cast<const Params<T> *>(vp);
    constexpr bool CPLX = same_t<T, float2>::value;
    TcPlan pl;
    if (!tc_plan(CPLX, (int)sizeof(T), p.m, p.n, p.k, B0, p.batch, pl)) return cudaErrorNotSupported;
    p.P = pl.P;
    p.S = pl.S | (pl.NU << 8) | (pl.CS << 16);
    p.ntiles = pl.ntiles;
    auto kern = &tc_kernel<T, OPA, OPB, B0>;
    const int grid = grid_for((const void *)kern, TC_NT, pl.smem, pl.ntiles);
    return launch_pdl(kern, grid, TC_NT, pl.smem, st, p);
}

}  // namespace tx
