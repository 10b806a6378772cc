// tx_common.cuh -- scalar types, the paper's entry-wise functors, and the sm_100a
// PTX wrappers (bulk async copies, mbarriers, cp.async) used by the kernels.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#else  // NVRTC (runtime specialisation, tx_jit.cu): no host headers
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#endif

namespace tx {

template <class A, class B> struct same_t { static constexpr bool value = false; };
template <class A> struct same_t<A, A> { static constexpr bool value = true; };

// Operation codes for op(X).  For real types 'C' maps to OP_T.
enum { OP_N = 0, OP_T = 1, OP_C = 2 };

// Path codes reported by tx_last_path() (include/txgemm.h).
enum { PATH_NONE = 0, PATH_BULK = 1, PATH_GATHER = 2, PATH_PTR = 3, PATH_SCALE = 4,
       PATH_DIRECT = 5, PATH_TC = 6, PATH_TAIL = 16, PATH_JIT = 32 };

template <class T> struct is_cplx { static constexpr bool value = false; };
template <> struct is_cplx<float2> { static constexpr bool value = true; };
template <> struct is_cplx<double2> { static constexpr bool value = true; };

// --------------------------------------------------------------------------
// Entry-wise arithmetic.  acc += op(a) * op(b) with the conjugations folded into
// the FMA operand signs (compile-time), i.e. the paper's unary_a / unary_b
// functors (identity / conjugate) applied without extra
// instructions.  Complex: 4-multiply form.
// --------------------------------------------------------------------------
template <bool CA, bool CB>
__device__ __forceinline__ void mac(float &acc, float a, float b) { acc = fmaf(a, b, acc); }
template <bool CA, bool CB>
__device__ __forceinline__ void mac(double &acc, double a, double b) { acc = fma(a, b, acc); }
template <bool CA, bool CB>
__device__ __forceinline__ void mac(float2 &acc, float2 a, float2 b)
{
    // re += ar*br - (sa*ai)*(sb*bi);  im += ar*(sb*bi) + (sa*ai)*br
    constexpr float sab = (CA != CB) ? 1.f : -1.f;  // -(sa*sb)
    constexpr float sb = CB ? -1.f : 1.f, sa = CA ? -1.f : 1.f;
#ifdef TX_FFMA2
    // sm_100 packed fp32 FMA (FFMA2; build with -DTX_FFMA2).  An interleaved gate A/B over
    // all 288 c instances measured no net gain (median ratio 1.002, 79 faster / 68 slower by
    // > 2 %; profiles/r02s3_ffma2_ab/): ncu (c13 beta = 0) shows issue 69 % -> 56 % but the
    // FMA pipe 48 % -> 52 % and the same duration -- the kernel is latency / occupancy bound
    // (16 warps per SM, per-tile barrier), not issue bound.  Kept as an option.
    // The same two fmas per component, same operand products, same order (re: ar*br, then
    // (sab*ai)*bi; im: ar*(sb*bi), then (sa*ai)*br; signs moved between factors are exact),
    // so results are bitwise those of the scalar chain below, with half the FMA instructions;
    // ar and sa*ai are broadcast operands, free in FFMA2.
    const float2 bs = make_float2(sa * sab * b.y, b.x);  // (sa*ai) * bs = (sab*ai*bi, sa*ai*br)
    acc = __ffma2_rn(make_float2(a.x, a.x), make_float2(b.x, sb * b.y), acc);
    acc = __ffma2_rn(make_float2(sa * a.y, sa * a.y), bs, acc);
#else
    acc.x = fmaf(a.x, b.x, acc.x);
    acc.x = fmaf(sab * a.y, b.y, acc.x);
    acc.y = fmaf(a.x, sb * b.y, acc.y);
    acc.y = fmaf(sa * a.y, b.x, acc.y);
#endif
}
template <bool CA, bool CB>
__device__ __forceinline__ void mac(double2 &acc, double2 a, double2 b)
{
    constexpr double sab = (CA != CB) ? 1.0 : -1.0;
    constexpr double sb = CB ? -1.0 : 1.0, sa = CA ? -1.0 : 1.0;
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(sab * a.y, b.y, acc.x);
    acc.y = fma(a.x, sb * b.y, acc.y);
    acc.y = fma(sa * a.y, b.x, acc.y);
}

template <class T> __host__ __device__ __forceinline__ T zero();
template <> __host__ __device__ __forceinline__ float zero<float>() { return 0.f; }
template <> __host__ __device__ __forceinline__ double zero<double>() { return 0.0; }
template <> __host__ __device__ __forceinline__ float2 zero<float2>() { return make_float2(0.f, 0.f); }
template <> __host__ __device__ __forceinline__ double2 zero<double2>() { return make_double2(0.0, 0.0); }

__device__ __forceinline__ bool is_zero(float v) { return v == 0.f; }
__device__ __forceinline__ bool is_zero(double v) { return v == 0.0; }
__device__ __forceinline__ bool is_zero(float2 v) { return v.x == 0.f && v.y == 0.f; }
__device__ __forceinline__ bool is_zero(double2 v) { return v.x == 0.0 && v.y == 0.0; }
__device__ __forceinline__ bool is_one(float v) { return v == 1.f; }
__device__ __forceinline__ bool is_one(double v) { return v == 1.0; }
__device__ __forceinline__ bool is_one(float2 v) { return v.x == 1.f && v.y == 0.f; }
__device__ __forceinline__ bool is_one(double2 v) { return v.x == 1.0 && v.y == 0.0; }

// y = a*x (axpby with b == 0: y is never read -- the paper's a1b0 generalised
// to any alpha) and y = a*x + b*y.
__device__ __forceinline__ float ax(float a, float x) { return a * x; }
__device__ __forceinline__ double ax(double a, double x) { return a * x; }
__device__ __forceinline__ float2 ax(float2 a, float2 x)
{
    return make_float2(fmaf(a.x, x.x, -a.y * x.y), fmaf(a.x, x.y, a.y * x.x));
}
__device__ __forceinline__ double2 ax(double2 a, double2 x)
{
    return make_double2(fma(a.x, x.x, -a.y * x.y), fma(a.x, x.y, a.y * x.x));
}
__device__ __forceinline__ float axpby(float a, float x, float b, float y) { return fmaf(b, y, a * x); }
__device__ __forceinline__ double axpby(double a, double x, double b, double y) { return fma(b, y, a * x); }
__device__ __forceinline__ float2 axpby(float2 a, float2 x, float2 b, float2 y)
{
    float2 r = ax(a, x);
    r.x = fmaf(b.x, y.x, r.x);
    r.x = fmaf(-b.y, y.y, r.x);
    r.y = fmaf(b.x, y.y, r.y);
    r.y = fmaf(b.y, y.x, r.y);
    return r;
}
__device__ __forceinline__ double2 axpby(double2 a, double2 x, double2 b, double2 y)
{
    double2 r = ax(a, x);
    r.x = fma(b.x, y.x, r.x);
    r.x = fma(-b.y, y.y, r.x);
    r.y = fma(b.x, y.y, r.y);
    r.y = fma(b.y, y.x, r.y);
    return r;
}

// --------------------------------------------------------------------------
// PTX wrappers (sm_90+/sm_100a): mbarrier, 1-D bulk async copies (TMA engine,
// SASS UBLKCP), async-proxy fence, and element-granular cp.async (LDGSTS).
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// plain arrive (release): a consumer warp's "stage consumed" signal
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TX_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TX_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// L2 eviction policy for streamed operands: each byte is used exactly once.
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// global -> shared bulk copy, completion counted on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes,
                                         uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// global -> shared tensor copy (TMA, SASS UTMALDG) of one box of a 2-D / 3-D
// tensor map, completion counted on an mbarrier.  tmap: generic address of a
// 128-byte tensor map in parameter space (__grid_constant__ kernel argument).
// The full box is always written (out-of-bounds rows are zero-filled), so the
// transaction count of a box is its full size.
__device__ __forceinline__ void tma_g2s_2d(void *sdst, const void *tmap, int c0, int c1,
                                           uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(sdst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tma_g2s_3d(void *sdst, const void *tmap, int c0, int c1, int c2,
                                           uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(sdst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// shared -> global bulk copy, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, uint32_t bytes,
                                         uint64_t pol)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait()
{
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Make this thread's generic-proxy shared-memory writes visible to the async
// proxy (required before a bulk store reads them).
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Element-granular async global -> shared copy (LDGSTS), 4/8/16 bytes.
template <int BYTES>
__device__ __forceinline__ void cp_async(void *sdst, const void *gsrc)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(sdst)), "l"(gsrc),
                 "n"(BYTES)
                 : "memory");
}
// 16-byte async copy that bypasses L1 (streamed data).
__device__ __forceinline__ void cp_async16_cg(void *sdst, const void *gsrc)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch (sm_90+): wait until the preceding grid in the
// stream has completed and its memory is visible (placed before the first
// global access), and allow the next grid to be scheduled early.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace tx
