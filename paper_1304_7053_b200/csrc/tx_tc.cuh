// tx_tc.cuh -- 5th-generation tensor-core (tcgen05, kind::tf32) path for the
// single-precision types (s, c) at the sizes beyond 16 where the FP32 FMA pipe,
// not HBM, bounds the CUDA-core kernels ("can be easily extended to larger
// sizes").
//
// Arithmetic: split-TF32 ("3xTF32").  Each fp32 operand x is split into
//   hi = rna_tf32(x),  lo = rna_tf32(x - hi)            (x - hi is exact in fp32)
// and  C^p = alpha * (A_hi B_lo + A_lo B_hi + A_hi B_hi) + beta * C^p,
// the three products accumulated in fp32 in TMEM by tcgen05.mma (the dropped
// A_lo B_lo term and the rounding of lo are O(2^-22) relative to |a||b|).
// Integer-valued inputs (|x| < 2^11) have lo = 0 and exact products, so the
// result is exact whenever the true sums are (bit-exact tests).
//
// Complex (c) in real form, rows interleaved (re, im):
//   X = [Ar_0; Ai_0; Ar_1; Ai_1; ...],  Y = [-Ai_0; Ar_0; -Ai_1; Ar_1; ...]   (2m x k)
//   D = X Br + Y Bi  ->  D[2i] = Re C_i.,  D[2i+1] = Im C_i.                 (2m x n)
// with Ai -> -Ai for op(A) = 'C' and Bi -> -Bi for op(B) = 'C'.
//
// Per CTA (persistent, 256 threads): thread 0 streams packed tiles of P pairs
// into an S-stage mbarrier ring with 1-D bulk copies (as bulk_kernel does); all
// threads split each pair's operands into hi/lo K-major 128-byte-swizzled
// canonical layouts in one of two operand buffers ("transform"); thread 0
// issues the MMAs (M = 128, N = roundup(n, 16), K = 8 per instruction) into one
// of two TMEM accumulators and commits them to mbarriers; while the tensor core
// runs, the threads transform the next pair and run the epilogue of the
// previous one (tcgen05.ld -> alpha/beta -> st.global).  Rows of the M = 128
// operand beyond the matrix read whatever follows in shared memory: they only
// produce accumulator rows that are never read.  K is padded with zeros.
#pragma once
#include "tx_kernels.cuh"

namespace tx {

template <class T> struct TcOk { static constexpr bool value = false; };
template <> struct TcOk<float> { static constexpr bool value = true; };
template <> struct TcOk<float2> { static constexpr bool value = true; };

constexpr int TC_NT = 256;             // 8 warps
constexpr int TC_SLACK = 16384;        // over-read of the last M = 128 operand
constexpr int TC_TMEM_COLS = 128;      // two accumulators of N <= 64 columns

// Shared-memory layout of one operand unit (one K-block of <= 32 elements).
//   real:    [A_hi | A_lo | B_hi | B_lo]            A: ar rows, B: N rows, 128 B each
//   complex: [X_hi | Y_hi | X_lo | Y_lo | Br_hi | Bi_hi | Br_lo | Bi_lo]
struct TcGeom {
    int ar;      // rows of an A-side array (roundup(m, 8) real, roundup(2m, 8) complex)
    int N;       // MMA N = roundup(n, 16)
    int KB;      // K-blocks of 32 elements per pair (complex: k <= 32 -> 1)
    int K8;      // roundup(k, 8)
    int abytes;  // one A-side array
    int bbytes;  // one B-side array
    int unit;    // one operand unit
};

__host__ __device__ inline TcGeom tc_geom(bool cplx, int m, int n, int k)
{
    TcGeom g;
    g.ar = cplx ? ((2 * m + 7) & ~7) : ((m + 7) & ~7);
    g.N = (n + 15) & ~15;
    g.K8 = (k + 7) & ~7;
    g.KB = (k + 31) / 32;
    g.abytes = g.ar * 128;
    g.bbytes = g.N * 128;
    g.unit = cplx ? 4 * g.abytes + 4 * g.bbytes : 2 * g.abytes + 2 * g.bbytes;
    return g;
}

// byte offset of element (r, kk), kk < 32, in a K-major SW128 array: 8-row groups
// 1024 B apart, 16-byte chunk c of row r at chunk c ^ (r mod 8).
__device__ __forceinline__ uint32_t tc_off(int r, int kk)
{
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((kk >> 2) ^ r) & 7) << 4));
}

__device__ __forceinline__ float tf32_rna(float x)
{
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return __uint_as_float(u);
}

// hi / lo parts of 4 values -> two 16-byte shared stores
__device__ __forceinline__ void tc_put4(unsigned char *hi, unsigned char *lo, uint32_t off, float v0,
                                        float v1, float v2, float v3)
{
    const float h0 = tf32_rna(v0), h1 = tf32_rna(v1), h2 = tf32_rna(v2), h3 = tf32_rna(v3);
    *reinterpret_cast<float4 *>(hi + off) = make_float4(h0, h1, h2, h3);
    *reinterpret_cast<float4 *>(lo + off) =
        make_float4(tf32_rna(v0 - h0), tf32_rna(v1 - h1), tf32_rna(v2 - h2), tf32_rna(v3 - h3));
}

// Shared-memory matrix descriptor (tcgen05): K-major, 128-byte swizzle, SBO = 1024.
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: kind::tf32, fp32 accumulator, both operands K-major, M = 128.
__device__ __forceinline__ uint32_t tc_idesc(int N)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
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

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 8 accumulator columns of this warp's 32 TMEM lanes (lane = D row)
__device__ __forceinline__ void tc_ld8(uint32_t taddr, float (&v)[8])
{
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}

// ---------------------------------------------------------------- transform
// Real: op(A) (m x k) and op(B) (k x n) of one pair, K-block kb, into hi/lo
// K-major arrays.  Thread order per array: rows fastest when the stored matrix
// is contiguous along the rows (conflict-free reads and swizzled stores),
// 16-byte chunks fastest when it is contiguous along K.
template <int OPA, int OPB>
__device__ __forceinline__ void tc_transform_real(const float *__restrict__ sA,
                                                  const float *__restrict__ sB, unsigned char *u,
                                                  const TcGeom &g, int m, int n, int k, int kb)
{
    const int tid = threadIdx.x;
    const int k0 = kb * 32;
    const int kw = min(32, g.K8 - k0);  // multiple of 8
    const int KC = kw >> 2;             // 16-byte chunks per row
    unsigned char *ahi = u, *alo = u + g.abytes, *bhi = u + 2 * g.abytes, *blo = bhi + g.bbytes;
    const bool vec = (k & 3) == 0;
    // A: element (i, l) = OPA == N ? sA[i + m*l] : sA[l + k*i]
    for (int w = tid; w < m * KC; w += TC_NT) {
        int i, c;
        if (OPA == OP_N) { i = w % m; c = w / m; } else { c = w % KC; i = w / KC; }
        const int l = k0 + 4 * c;
        float v[4];
        if (OPA != OP_N && vec && l + 3 < k) {
            const float4 t = *reinterpret_cast<const float4 *>(sA + l + (long long)k * i);
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                v[e] = (l + e < k) ? (OPA == OP_N ? sA[i + m * (l + e)] : sA[(l + e) + k * i]) : 0.f;
        }
        tc_put4(ahi, alo, tc_off(i, 4 * c), v[0], v[1], v[2], v[3]);
    }
    // B: element (l, j) = OPB == N ? sB[l + k*j] : sB[j + n*l]; row j of the operand
    for (int w = tid; w < n * KC; w += TC_NT) {
        int j, c;
        if (OPB == OP_N) { c = w % KC; j = w / KC; } else { j = w % n; c = w / n; }
        const int l = k0 + 4 * c;
        float v[4];
        if (OPB == OP_N && vec && l + 3 < k) {
            const float4 t = *reinterpret_cast<const float4 *>(sB + l + (long long)k * j);
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                v[e] = (l + e < k) ? (OPB == OP_N ? sB[(l + e) + k * j] : sB[j + n * (l + e)]) : 0.f;
        }
        tc_put4(bhi, blo, tc_off(j, 4 * c), v[0], v[1], v[2], v[3]);
    }
}

// Complex: X, Y (rows 2i + e) and Br, Bi (rows j), k <= 32 (one K-block).
template <int OPA, int OPB>
__device__ __forceinline__ void tc_transform_cplx(const float2 *__restrict__ sA,
                                                  const float2 *__restrict__ sB, unsigned char *u,
                                                  const TcGeom &g, int m, int n, int k)
{
    const int tid = threadIdx.x;
    const int KC = g.K8 >> 2;
    unsigned char *xhi = u, *yhi = u + g.abytes, *xlo = u + 2 * g.abytes, *ylo = u + 3 * g.abytes;
    unsigned char *rhi = u + 4 * g.abytes, *ihi = rhi + g.bbytes, *rlo = ihi + g.bbytes,
                  *ilo = rlo + g.bbytes;
    constexpr float sa = OPA == OP_C ? -1.f : 1.f, sb = OPB == OP_C ? -1.f : 1.f;
    const bool vec = (k & 1) == 0;
    // A: item (i, e, c); e = 0 -> X row 2i <- ar, Y row 2i+1 <- ar;
    //                    e = 1 -> X row 2i+1 <- sa*ai, Y row 2i <- -sa*ai
    for (int w = tid; w < 2 * m * KC; w += TC_NT) {
        int i, e, c;
        if (OPA == OP_N) { e = w & 1; i = (w >> 1) % m; c = (w >> 1) / m; }
        else { c = w % KC; e = (w / KC) & 1; i = (w / KC) >> 1; }
        const int l = 4 * c;
        float2 a[4];
        if (OPA != OP_N && vec && l + 3 < k) {
            const float4 *p = reinterpret_cast<const float4 *>(sA + l + (long long)k * i);
            const float4 t0 = p[0], t1 = p[1];
            a[0] = make_float2(t0.x, t0.y); a[1] = make_float2(t0.z, t0.w);
            a[2] = make_float2(t1.x, t1.y); a[3] = make_float2(t1.z, t1.w);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                a[q] = (l + q < k) ? (OPA == OP_N ? sA[i + m * (l + q)] : sA[(l + q) + k * i])
                                   : make_float2(0.f, 0.f);
        }
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = e ? sa * a[q].y : a[q].x;
        const int rx = 2 * i + e, ry = 2 * i + 1 - e;
        tc_put4(xhi, xlo, tc_off(rx, l), v[0], v[1], v[2], v[3]);
        if (e)
            tc_put4(yhi, ylo, tc_off(ry, l), -v[0], -v[1], -v[2], -v[3]);
        else
            tc_put4(yhi, ylo, tc_off(ry, l), v[0], v[1], v[2], v[3]);
    }
    // B: item (j, c): Br row j <- br, Bi row j <- sb*bi
    for (int w = tid; w < n * KC; w += TC_NT) {
        int j, c;
        if (OPB == OP_N) { c = w % KC; j = w / KC; } else { j = w % n; c = w / n; }
        const int l = 4 * c;
        float2 b[4];
        if (OPB == OP_N && vec && l + 3 < k) {
            const float4 *p = reinterpret_cast<const float4 *>(sB + l + (long long)k * j);
            const float4 t0 = p[0], t1 = p[1];
            b[0] = make_float2(t0.x, t0.y); b[1] = make_float2(t0.z, t0.w);
            b[2] = make_float2(t1.x, t1.y); b[3] = make_float2(t1.z, t1.w);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                b[q] = (l + q < k) ? (OPB == OP_N ? sB[(l + q) + k * j] : sB[j + n * (l + q)])
                                   : make_float2(0.f, 0.f);
        }
        const uint32_t off = tc_off(j, l);
        tc_put4(rhi, rlo, off, b[0].x, b[1].x, b[2].x, b[3].x);
        tc_put4(ihi, ilo, off, sb * b[0].y, sb * b[1].y, sb * b[2].y, sb * b[3].y);
    }
}

// MMAs of one operand unit into the accumulator at `tmem` (thread 0).
template <bool CPLX>
__device__ __forceinline__ void tc_issue(uint32_t ubase, const TcGeom &g, int kb, uint32_t tmem)
{
    const uint32_t id = tc_idesc(g.N);
    const int ksteps = min(32, g.K8 - kb * 32) >> 3;
    for (int s = 0; s < ksteps; ++s) {
        const uint32_t ko = s * 32;  // 8 tf32 = 32 bytes along K inside the swizzle atom
        const uint32_t first = (kb == 0 && s == 0) ? 0u : 1u;
        if constexpr (!CPLX) {
            const uint32_t ahi = ubase, alo = ahi + g.abytes, bhi = ubase + 2 * g.abytes,
                           blo = bhi + g.bbytes;
            tc_mma(tmem, tc_desc(ahi + ko), tc_desc(blo + ko), id, first);
            tc_mma(tmem, tc_desc(alo + ko), tc_desc(bhi + ko), id, 1u);
            tc_mma(tmem, tc_desc(ahi + ko), tc_desc(bhi + ko), id, 1u);
        } else {
            const uint32_t xhi = ubase, yhi = xhi + g.abytes, xlo = yhi + g.abytes,
                           ylo = xlo + g.abytes;
            const uint32_t rhi = ubase + 4 * g.abytes, ihi = rhi + g.bbytes, rlo = ihi + g.bbytes,
                           ilo = rlo + g.bbytes;
            tc_mma(tmem, tc_desc(xhi + ko), tc_desc(rlo + ko), id, first);
            tc_mma(tmem, tc_desc(xlo + ko), tc_desc(rhi + ko), id, 1u);
            tc_mma(tmem, tc_desc(yhi + ko), tc_desc(ilo + ko), id, 1u);
            tc_mma(tmem, tc_desc(ylo + ko), tc_desc(ihi + ko), id, 1u);
            tc_mma(tmem, tc_desc(xhi + ko), tc_desc(rhi + ko), id, 1u);
            tc_mma(tmem, tc_desc(yhi + ko), tc_desc(ihi + ko), id, 1u);
        }
    }
}

// Epilogue of one pair: accumulator rows -> alpha/beta -> C (column-major, ld = m).
// Warp w reads TMEM lanes 32*(w%4).. (rows), warps w and w+4 split the columns.
template <class T, bool B0>
__device__ __forceinline__ void tc_epilogue(uint32_t tacc, const T *__restrict__ sC,
                                            T *__restrict__ gC, int m, int n, const TcGeom &g,
                                            T alpha, T beta)
{
    constexpr bool CPLX = same_t<T, float2>::value;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb = warp & 3, half = warp >> 2;
    const int rows = CPLX ? 2 * m : m;
    if (rb * 32 >= rows) return;  // warp-uniform
    const int n8 = (n + 7) & ~7;
    const int nh = ((n8 >> 3) + 1) >> 1;  // column chunks of 8 in the first half
    const int c_lo = half ? nh : 0, c_hi = half ? (n8 >> 3) : nh;
    const int r = rb * 32 + lane;
    const uint32_t lane_addr = tacc + ((uint32_t)(rb * 32) << 16);
    for (int cc = c_lo; cc < c_hi; ++cc) {
        float v[8];
        tc_ld8(lane_addr + cc * 8, v);
        if constexpr (!CPLX) {
            if (r < m) {
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int j = cc * 8 + t;
                    if (j < n) {
                        const long long o = r + (long long)m * j;
                        gC[o] = B0 ? ax(alpha, v[t]) : axpby(alpha, v[t], beta, sC[o]);
                    }
                }
            }
        } else {
            const int i = r >> 1, e = r & 1;
#pragma unroll
            for (int t = 0; t < 8; t += 2) {
                const float send = e ? v[t] : v[t + 1];
                const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                const int j = cc * 8 + t + e;
                if (i < m && j < n) {
                    const float2 x = e ? make_float2(recv, v[t + 1]) : make_float2(v[t], recv);
                    const long long o = i + (long long)m * j;
                    gC[o] = B0 ? ax(alpha, x) : axpby(alpha, x, beta, sC[o]);
                }
            }
        }
    }
}

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
    const int P = p.P, S = p.S;
    const int ES = (int)sizeof(T);
    const int offB = P * SA * ES, offC = offB + P * SB * ES;
    const int stage_bytes = ((offC + (B0 ? 0 : P * SC * ES)) + 1023) & ~1023;
    unsigned char *base = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char *ubuf = base + (long long)S * stage_bytes;  // two operand units
    uint64_t *bars = reinterpret_cast<uint64_t *>(ubuf + 2 * g.unit + TC_SLACK);
    uint64_t *full = bars, *opfree = bars + S, *accfull = bars + S + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + S + 4);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;
    const uint64_t pol = policy_evict_first();

    if (tid == 0) {
        for (int s = 0; s < S + 4; ++s) mbar_init(&bars[s], 1);
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
    const T alpha = p.alpha, beta = p.beta;

    auto issue = [&](int i) {  // local tile i -> stage i % S (thread 0)
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        unsigned char *st = base + (long long)(i % S) * stage_bytes;
        uint64_t *bar = &full[i % S];
        const uint32_t ba = np * SA * ES, bb = np * SB * ES, bc = B0 ? 0u : np * SC * ES;
        mbar_arrive_expect_tx(bar, ba + bb + bc);
        bulk_g2s(st, p.A + pair0 * SA, ba, bar, pol);
        bulk_g2s(st + offB, p.B + pair0 * SB, bb, bar, pol);
        if (!B0) bulk_g2s(st + offC, p.C + pair0 * SC, bc, bar, pol);
    };
    if (tid == 0)
        for (int i = 0; i < S && i < my_tiles; ++i) issue(i);

    int u = 0;                         // operand units transformed so far
    int pp = 0;                        // pairs issued so far
    int pend_tile = -1, pend_q = 0;    // pair whose epilogue is pending
    auto epilogue = [&](int tile, int q, int ppi) {
        mbar_wait(&accfull[ppi & 1], (ppi >> 1) & 1);
        tc_fence_after();
        const long long pair0 = (blockIdx.x + (long long)tile * G) * P;
        const unsigned char *st = base + (long long)(tile % S) * stage_bytes;
        const T *sC = reinterpret_cast<const T *>(st + offC) + (long long)q * SC;
        tc_epilogue<T, B0>(tmem + (uint32_t)((ppi & 1) * 64), sC, p.C + (pair0 + q) * SC, m, n, g,
                           alpha, beta);
        tc_fence_before();
    };

    for (int i = 0; i < my_tiles; ++i) {
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        const unsigned char *st = base + (long long)(i % S) * stage_bytes;
        mbar_wait(&full[i % S], (i / S) & 1);
        for (int q = 0; q < np; ++q) {
            const T *sA = reinterpret_cast<const T *>(st) + (long long)q * SA;
            const T *sB = reinterpret_cast<const T *>(st + offB) + (long long)q * SB;
            for (int kb = 0; kb < KB; ++kb) {
                const int b = u & 1;
                if (u >= 2) mbar_wait(&opfree[b], ((u >> 1) - 1) & 1);  // MMAs of unit u-2 done
                unsigned char *ub = ubuf + b * g.unit;
                if constexpr (CPLX)
                    tc_transform_cplx<OPA, OPB>(sA, sB, ub, g, m, n, k);
                else
                    tc_transform_real<OPA, OPB>(sA, sB, ub, g, m, n, k, kb);
                fence_proxy_async_smem();
                tc_fence_before();
                __syncthreads();
                if (tid == 0) {
                    tc_fence_after();
                    tc_issue<CPLX>(smem_u32(ub), g, kb, tmem + (uint32_t)((pp & 1) * 64));
                    tc_commit(&opfree[b]);
                    if (kb == KB - 1) tc_commit(&accfull[pp & 1]);
                }
                ++u;
            }
            if (pend_tile >= 0) {
                epilogue(pend_tile, pend_q, pp - 1);
                if (pend_tile != i) {  // the previous tile is fully consumed: refill its stage
                    __syncthreads();
                    if (tid == 0 && pend_tile + S < my_tiles) issue(pend_tile + S);
                }
            }
            pend_tile = i;
            pend_q = q;
            ++pp;
        }
    }
    if (pend_tile >= 0) epilogue(pend_tile, pend_q, pp - 1);
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(TC_TMEM_COLS)
                     : "memory");
    }
}

}  // namespace tx

namespace tx {

// Host plan of the tensor-core kernel: P (a multiple of the 16-byte alignment
// unit) pairs per stage and S stages such that (S - 1) stages in flight cover
// >= 48 KB (the HBM latency-bandwidth product of one SM), within 227 KB.
struct TcPlan {
    int P, S, smem, ntiles;
};

inline int tc_smem_bytes(bool cplx, int es, int m, int n, int k, bool b0, int P, int S)
{
    const TcGeom g = tc_geom(cplx, m, n, k);
    const int stage = ((P * (m * k + k * n + (b0 ? 0 : m * n)) * es) + 1023) & ~1023;
    return 1024 + S * stage + 2 * g.unit + TC_SLACK + (S + 4) * 8 + 16;
}

inline bool tc_plan(bool cplx, int es, int m, int n, int k, bool b0, int unit, int batch, TcPlan &pl)
{
    const int pair_bytes = (m * k + k * n + (b0 ? 0 : m * n)) * es;
    int bestP = 0, bestS = 0;
    long long best_flight = -1;
    for (int P = unit; P <= 64 * unit; P += unit) {
        int S = 0;
        for (int s = 4; s >= 2; --s)
            if (tc_smem_bytes(cplx, es, m, n, k, b0, P, s) <= SMEM_MAX_BYTES) {
                S = s;
                break;
            }
        if (S == 0) break;
        const long long flight = (long long)(S - 1) * P * pair_bytes;
        if (flight > best_flight) {
            best_flight = flight;
            bestP = P;
            bestS = S;
        }
        if (flight >= 48 * 1024) break;
    }
    if (bestP == 0) return false;
    // keep every SM busy for small batches
    const int sms = num_sms();
    while (bestP > unit && (long long)(batch + bestP - 1) / bestP < sms) bestP -= unit;
    pl.P = bestP;
    pl.S = bestS;
    pl.smem = tc_smem_bytes(cplx, es, m, n, k, b0, pl.P, pl.S);
    pl.ntiles = (batch + pl.P - 1) / pl.P;
    return true;
}

// Launch (packed layout, 16-byte aligned, batch a multiple of `unit` = p.P on entry).
template <class T, int OPA, int OPB, bool B0>
cudaError_t launch_tc(const void *vp, cudaStream_t st)
{
    Params<T> p = *static_cast<const Params<T> *>(vp);
    constexpr bool CPLX = same_t<T, float2>::value;
    TcPlan pl;
    if (!tc_plan(CPLX, (int)sizeof(T), p.m, p.n, p.k, B0, p.P, p.batch, pl))
        return cudaErrorNotSupported;
    p.P = pl.P;
    p.S = pl.S;
    p.ntiles = pl.ntiles;
    auto kern = &tc_kernel<T, OPA, OPB, B0>;
    const int grid = grid_for((const void *)kern, TC_NT, pl.smem, pl.ntiles);
    return launch_pdl(kern, grid, TC_NT, pl.smem, st, p);
}

}  // namespace tx
