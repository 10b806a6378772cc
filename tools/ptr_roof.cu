// tools/ptr_roof.cu -- measurement tool (NOT the product): the memory system's
// throughput for the access pattern of a pointer-array batch, with no GEMM.
//
// For pair p it reads the bytes of A^p, B^p (and C^p when read_c) through the
// pointer arrays and writes C^p (every byte), exactly the algorithmic traffic of
// one batched-GEMM call on that layout, with a trivial "computation" (C^p gets a
// copy of A^p's first 16 bytes repeated, so nothing can be elided).  One warp per
// pair, 16-byte accesses (4-byte when the matrix size or address forbids),
// grid-stride over the batch with 2 pairs per warp in flight.  The ratio
// (GEMM time / this time) is how close the GEMM kernel is to the pattern's own
// roof: for permuted pointers to small matrices that roof is well below the
// streaming copy bandwidth (DRAM row locality is lost and sectors are shared by
// neighbouring matrices that are fetched at different times).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o tools/libptrroof.so tools/ptr_roof.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint4 ldcs16(const void *p)
{
    uint4 r;
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// bytes of each matrix; all three pointer arrays hold byte addresses
__global__ void __launch_bounds__(256) ptr_roof_kernel(const char *const *Ap, const char *const *Bp,
                                                       char *const *Cp, int ba, int bb, int bc,
                                                       int read_c, long long batch,
                                                       unsigned long long *sink)
{
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    for (long long p = warp; p < batch; p += nwarps) {
        const char *a = Ap[p], *b = Bp[p];
        char *c = Cp[p];
        const bool v16 = ((((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15) == 0) &&
                         (ba % 16 == 0) && (bb % 16 == 0) && (bc % 16 == 0);
        uint4 first = make_uint4(0, 0, 0, 0);
        if (v16) {
            for (int o = lane * 16; o < ba; o += 512) {
                const uint4 v = ldcs16(a + o);
                acc ^= v.x ^ v.w;
                if (o == 0) first = v;
            }
            for (int o = lane * 16; o < bb; o += 512) {
                const uint4 v = ldcs16(b + o);
                acc ^= v.y;
            }
            if (read_c)
                for (int o = lane * 16; o < bc; o += 512) {
                    const uint4 v = ldcs16(c + o);
                    acc ^= v.z;
                }
            first.x = __shfl_sync(0xffffffffu, first.x, 0);
            first.y = __shfl_sync(0xffffffffu, first.y, 0);
            first.z = __shfl_sync(0xffffffffu, first.z, 0);
            first.w = __shfl_sync(0xffffffffu, first.w ^ (acc & 1u), 0);
            for (int o = lane * 16; o < bc; o += 512) *reinterpret_cast<uint4 *>(c + o) = first;
        } else {
            for (int o = lane * 4; o < ba; o += 128) acc ^= *reinterpret_cast<const unsigned *>(a + o);
            for (int o = lane * 4; o < bb; o += 128) acc ^= *reinterpret_cast<const unsigned *>(b + o);
            if (read_c)
                for (int o = lane * 4; o < bc; o += 128) acc ^= *reinterpret_cast<const unsigned *>(c + o);
            const unsigned f = __shfl_sync(0xffffffffu, acc, 0);
            for (int o = lane * 4; o < bc; o += 128) *reinterpret_cast<unsigned *>(c + o) = f;
        }
    }
    if (acc == 0x9e3779b9u) atomicAdd(sink, 1ull);  // practically never; keeps the loads live
}

extern "C" int ptr_roof(const void *Ap, const void *Bp, const void *Cp, int ba, int bb, int bc,
                        int read_c, long long batch, void *sink, int blocks, void *stream)
{
    ptr_roof_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        (const char *const *)Ap, (const char *const *)Bp, (char *const *)Cp, ba, bb, bc, read_c,
        batch, (unsigned long long *)sink);
    return (int)cudaGetLastError();
}
