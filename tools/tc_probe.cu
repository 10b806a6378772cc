// tc_probe.cu -- what tcgen05.mma kind::tf32 computes on this B200 (measurement tool).
//
// One CTA of 128 threads: A (128 x K) and B (N x K), both K-major, are written into
// shared memory in the 128-byte-swizzled canonical layout, one thread issues
// tcgen05.mma.cta_group::1.kind::tf32 (M = 128) over K in steps of 8, the four warps
// read the accumulator back with tcgen05.ld.32x32b and write D (128 x N, row-major).
// M = 64 or 128 (the M = 64 run reports where D's rows land in TMEM: row r of D in
// lane L of the output when D[L][*] holds row r's values).
// nsets = 1: D = A0 B0^T; nsets = 3: D = A0 B1^T + A1 B0^T + A0 B0^T (the 3xTF32 order
// with A0/B0 = hi, A1/B1 = lo parts), all into one accumulator.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o libtcprobe.so tc_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t su32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (r, k) (fp32) in a K-major SW128 operand whose K-blocks of 32
// elements are `rows * 128` bytes apart; 8-row groups 1024 B apart (SBO).
__device__ __forceinline__ uint32_t kmaj_off(int r, int k, int rows)
{
    const int kb = k >> 5, kk = k & 31;
    return kb * rows * 128 + (r >> 3) * 1024 + (r & 7) * 128 + ((((kk >> 2) ^ (r & 7)) & 7) << 4) +
           (kk & 3) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;             // LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;   // SBO: 8-row groups
    d |= (uint64_t)1 << 46;             // version (sm100)
    d |= (uint64_t)2 << 61;             // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ uint32_t idesc_tf32(int M, int N, int nega, int negb)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)nega << 13) | ((uint32_t)negb << 14) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1)
probe_kernel(const float *A0, const float *A1, const float *B0, const float *B1, float *D, int N,
             int K, int nsets, int M)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KB = (K + 31) / 32;
    unsigned char *sA0 = smem + ((1024u - (su32(smem) & 1023u)) & 1023u);
    unsigned char *sA1 = sA0 + KB * 128 * 128;
    unsigned char *sB0 = sA1 + KB * 128 * 128;
    unsigned char *sB1 = sB0 + KB * N * 128;
    for (int e = tid; e < 128 * K; e += 128) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<float *>(sA0 + kmaj_off(r, k, 128)) = A0[e];
        *reinterpret_cast<float *>(sA1 + kmaj_off(r, k, 128)) = A1[e];
    }
    for (int e = tid; e < N * K; e += 128) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<float *>(sB0 + kmaj_off(r, k, N)) = B0[e];
        *reinterpret_cast<float *>(sB1 + kmaj_off(r, k, N)) = B1[e];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t id = idesc_tf32(M, N, 0, 0);
        int first = 1;
        for (int s = 0; s < K / 8; ++s) {
            const uint32_t kb = s >> 2, kin = (s & 3) * 32;
            const uint32_t a0 = su32(sA0) + kb * 128 * 128 + kin, a1 = su32(sA1) + kb * 128 * 128 + kin;
            const uint32_t b0 = su32(sB0) + kb * N * 128 + kin, b1 = su32(sB1) + kb * N * 128 + kin;
            const uint64_t pa[3] = {sdesc(a0), sdesc(a1), sdesc(a0)};
            const uint64_t pb[3] = {sdesc(b1), sdesc(b0), sdesc(b0)};
            for (int t = (nsets == 3 ? 0 : 2); t < 3; ++t) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(pa[t]), "l"(pb[t]), "r"(id), "r"(first ? 0 : 1));
                first = 0;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            su32(&bar)));
    }
    // wait for the MMAs (parity 0)
    asm volatile(
        "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}\n" ::"r"(
            su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

}  // namespace

extern "C" int tc_probe(const float *A0, const float *A1, const float *B0, const float *B1, float *D,
                        int N, int K, int nsets, int M)
{
    const int KB = (K + 31) / 32;
    const size_t smem = (size_t)KB * 128 * (2 * 128 + 2 * N) + 1024;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_kernel<<<1, 128, smem>>>(A0, A1, B0, B1, D, N, K, nsets, M);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}
