// tx_jit.h -- runtime specialisation (NVRTC) of the batched-GEMM kernels: see tx_jit.cu.
#pragma once

#include <cuda.h>

#include <string>

#include "tx_dispatch.cuh"

namespace tx {

struct JitMap {
    int RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN, S, KB;
    int ASW = 0;  // gather instances: A copies placed in the swizzled layout (ASWG)
    int BSW = 0;  // ... and B copies (BSWG)
};

bool jit_available();
int jit_set_enabled(int on);
int jit_compiled_count();
CUfunction jit_function(const std::string &name_expr);
int jit_occupancy(CUfunction f, int nt, int smem);
cudaError_t jit_launch(CUfunction f, int grid, int nt, int smem, cudaStream_t st, void *params);
JitMap jit_mapping(int es, bool cplx, int m, int n, int k, int opa, int opb, bool b0,
                   bool global_c, bool asw_ok = false, bool bsw_ok = false);
std::string jit_map_string(const JitMap &mp);

template <class T> inline const char *type_name();
template <> inline const char *type_name<float>() { return "float"; }
template <> inline const char *type_name<double>() { return "double"; }
template <> inline const char *type_name<float2>() { return "float2"; }
template <> inline const char *type_name<double2>() { return "double2"; }

enum JitKind { JIT_BULK = 0, JIT_BULK_PTR = 1, JIT_GATHER = 2, JIT_GATHER_PTR = 3,
               JIT_GATHER_PTR16 = 4 };

// Launch the runtime-specialised kernel of `kind` for p (sizes static in the
// instance).  Returns cudaErrorNotSupported when JIT is unavailable so the
// caller can use an AOT kernel instead.
template <class T>
cudaError_t launch_jit(JitKind kind, Params<T> p, int opa, int opb, bool b0, cudaStream_t st,
                       int bcast = 0, bool devab = false)
{
    if (devab && kind == JIT_BULK_PTR) kind = JIT_GATHER_PTR16;  // no DEVAB bulk_ptr kernel
    if (!jit_available()) return cudaErrorNotSupported;
    const bool cplx = is_cplx<T>::value;
    const bool gather = kind == JIT_GATHER || kind == JIT_GATHER_PTR || kind == JIT_GATHER_PTR16;
    // swizzled A placement is possible in the gather kernels when a stored column of
    // op(A) = T/C spans whole 128-byte lines
    const bool asw_ok = gather && !devab && opa != OP_N && (p.k * (int)sizeof(T)) % 128 == 0;
    const bool bsw_ok = gather && !devab && opb == OP_N && (p.k * (int)sizeof(T)) % 128 == 0;
    JitMap mp = jit_mapping((int)sizeof(T), cplx, p.m, p.n, p.k, opa, opb, b0,
                            kind != JIT_BULK, asw_ok, bsw_ok);
    constexpr int NT = NT_DEFAULT;
    char head[256];
    const char *kname = kind == JIT_BULK ? "bulk_kernel"
                        : kind == JIT_BULK_PTR ? "bulk_ptr_kernel" : "gather_kernel";
    snprintf(head, sizeof(head), "&tx::%s<%s, %d, %d, %d, %d, %d, %s, ", kname, type_name<T>(),
             p.m, p.n, p.k, opa, opb, b0 ? "true" : "false");
    std::string expr = std::string(head) + jit_map_string(mp) + ", " + std::to_string(NT);
    if (gather) {  // <..., PTR, V16, DEVAB, ASWG, BSWG>
        expr += kind == JIT_GATHER ? ", false" : ", true";
        expr += kind == JIT_GATHER_PTR16 ? ", true" : ", false";
        expr += devab ? ", true" : ", false";
        expr += mp.ASW ? ", true" : ", false";
        expr += mp.BSW ? ", true" : ", false";
    }
    if (kind == JIT_BULK && (bcast || devab)) expr += ", " + std::to_string(bcast);
    if (kind == JIT_BULK && devab) expr += ", false, true";
    expr += ">";
    CUfunction f = jit_function(expr);
    if (!f) return cudaErrorNotSupported;
    Plan pl = plan_tiles(sizeof(T), p.m, p.n, p.k, b0, mp.RM, mp.RN, NT, p.batch, !gather,
                         gather ? GS : mp.S, mp.KB, kind == JIT_BULK ? bcast : 0);
    if (kind == JIT_GATHER_PTR || kind == JIT_GATHER_PTR16)
        gather_ptr_plan(pl, (int)sizeof(T), p.m, p.n, p.k, b0, p.batch);
    if (kind == JIT_BULK_PTR && pl.P > 128) {  // bulk_ptr_kernel: <= 4 pointer triples per lane
        pl.P = 128;
        pl.ntiles = (int)(((long long)p.batch + 127) / 128);
        const int SA = p.m * p.k, SB = p.k * p.n, SC = p.m * p.n;
        pl.smem = pl.S * 128 * (SA + SB + (b0 ? 0 : SC)) * (int)sizeof(T) + 8 * pl.S;
    }
    p.P = pl.P;
    p.S = pl.S;
    p.ntiles = pl.ntiles;
    long long grid = (long long)num_sms() * jit_occupancy(f, NT, pl.smem);
    const int cap = max_ctas_override();
    if (cap > 0 && grid > cap) grid = cap;
    if (grid > pl.ntiles) grid = pl.ntiles;
    if (grid < 1) grid = 1;
    return jit_launch(f, (int)grid, NT, pl.smem, st, &p);
}

}  // namespace tx
