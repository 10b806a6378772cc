// tc_trace.cu -- per-phase clock64 timeline of the tensor-core kernel's CTA 0 (measurement
// tool): producer issue, transform start/end, MMA start/committed, epilogue start/end per
// operand unit / pair.  Built with TC_TRACE so the kernel records tc_trace[event][index].
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_1304_7053_b200/csrc -shared -Xcompiler -fPIC -o tools/libtctrace.so tools/tc_trace.cu
#define TC_TRACE 1
#include "tx_dispatch.cuh"
#include "tx_tc.cuh"

namespace tx {
int num_sms()
{
    int d = 0, n = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
}
int max_ctas_override() { return 0; }
bool prepare_only() { return false; }
int tune_stages() { return 0; }
int tune_stage_bytes() { return 0; }
}  // namespace tx

template <class T, bool B0>
static int run(int m, int n, int k, int batch, void *A, void *B, void *C, unsigned long long *out,
               float *ms)
{
    tx::Params<T> p;
    memset(&p, 0, sizeof(p));
    p.A = (const T *)A;
    p.B = (const T *)B;
    p.C = (T *)C;
    p.m = m;
    p.n = n;
    p.k = k;
    p.lda = m;
    p.ldb = k;
    p.ldc = m;
    p.lda2 = (long long)m * k;
    p.ldb2 = (long long)k * n;
    p.ldc2 = (long long)m * n;
    p.batch = batch;
    p.P = 1;
    if constexpr (sizeof(T) == 4) {
        p.alpha = 1.f;
        p.beta = B0 ? 0.f : 0.5f;
    } else {
        p.alpha = make_float2(1.f, 0.f);
        p.beta = B0 ? make_float2(0.f, 0.f) : make_float2(0.5f, 0.f);
    }
    void *tr = nullptr;
    cudaGetSymbolAddress(&tr, tx::tc_trace);
    cudaMemset(tr, 0, sizeof(unsigned long long) * 8 * 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, 0);
    cudaError_t e = tx::launch_tc<T, 0, 0, B0>(&p, 0);
    if (e != cudaSuccess) return (int)e;
    cudaEventRecord(b, 0);
    e = cudaDeviceSynchronize();
    cudaEventElapsedTime(ms, a, b);
    if (e != cudaSuccess) return (int)e;
    cudaMemcpyFromSymbol(out, tx::tc_trace, sizeof(unsigned long long) * 8 * 256);
    return 0;
}

extern "C" int tc_trace_run(int cplx, int beta0, int m, int n, int k, int batch, void *A, void *B,
                            void *C, unsigned long long *out, float *ms)
{
    if (cplx) return beta0 ? run<float2, true>(m, n, k, batch, A, B, C, out, ms)
                           : run<float2, false>(m, n, k, batch, A, B, C, out, ms);
    return beta0 ? run<float, true>(m, n, k, batch, A, B, C, out, ms)
                 : run<float, false>(m, n, k, batch, A, B, C, out, ms);
}
