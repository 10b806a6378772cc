// tools/dmma_probe.cu -- measurement tool (NOT the product): what does the FP64
// tensor-core MMA (mma.sync m8n8k4 f64, SASS DMMA) compute, bit for bit?
// Each warp multiplies one 8x4 A by one 4x8 B onto an 8x8 C; the host compares
// D with candidate evaluation orders (sequential fused multiply-adds over k, ...).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o tools/libdmmaprobe.so tools/dmma_probe.cu
#include <cuda_runtime.h>

__global__ void dmma_probe_kernel(const double *A, const double *B, const double *C, double *D,
                                  int nwarps)
{
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= nwarps) return;
    const double *a = A + w * 32, *b = B + w * 32, *c = C + w * 64;
    // assumed fragment layouts (PTX m8n8k4 .f64): A row-major 8x4: a0 = A[g][t];
    // B column-major 4x8: b0 = B[t][g]; C/D 8x8: {c0, c1} = C[g][2t], C[g][2t+1]
    const int g = lane >> 2, t = lane & 3;
    const double a0 = a[g * 4 + t];
    const double b0 = b[t * 8 + g];
    const double c0 = c[g * 8 + 2 * t], c1 = c[g * 8 + 2 * t + 1];
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a0), "d"(b0), "d"(c0), "d"(c1));
    D[w * 64 + g * 8 + 2 * t] = d0;
    D[w * 64 + g * 8 + 2 * t + 1] = d1;
}

extern "C" int dmma_probe(const double *A, const double *B, const double *C, double *D, int nwarps)
{
    dmma_probe_kernel<<<(nwarps * 32 + 255) / 256, 256>>>(A, B, C, D, nwarps);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}

// Throughput: each warp runs `iters` x 8 independent DMMA (or 8 x 32 independent
// DFMA chains per thread-step); returns elapsed ms for a full-GPU launch.
__global__ void dmma_rate_kernel(double *out, int iters)
{
    double d[8][2];
    for (int q = 0; q < 8; ++q) d[q][0] = d[q][1] = threadIdx.x * 1e-3 + q;
    const double a = 1.0000001, b = 0.9999999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[q][0]), "+d"(d[q][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int q = 0; q < 8; ++q) s += d[q][0] + d[q][1];
    if (s == 123.456) out[0] = s;
}

__global__ void dfma_rate_kernel(double *out, int iters)
{
    double d[8];
    for (int q = 0; q < 8; ++q) d[q] = threadIdx.x * 1e-3 + q;
    const double a = 1.0000001, b = 0.9999999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 32; ++r)
#pragma unroll
            for (int q = 0; q < 8; ++q) d[q] = fma(a, d[q], b);
    }
    double s = 0;
    for (int q = 0; q < 8; ++q) s += d[q];
    if (s == 123.456) out[0] = s;
}

// flops per launch: dmma: blocks*warps*iters*8*(8*8*4*2); dfma: threads*iters*32*8*2
extern "C" float dmma_rate(int which, int blocks, int threads, int iters, double *out)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (which == 0) dmma_rate_kernel<<<blocks, threads>>>(out, iters);
        else dfma_rate_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}
