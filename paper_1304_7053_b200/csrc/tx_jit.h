// tx_jit.h -- runtime specialisation (NVRTC) of the batched-GEMM kernels: see tx_jit.cu.
#pragma once

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
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
    // bulk: the tile by a TMA tensor copy with the swizzle (ASW / BSW); gather: the
    // copies placed in the swizzled layout (ASWG / BSWG)
    // (bulk: k <= 16 only, so the 1024-byte stage alignment never pushes a plan past
    // the shared-memory limit)
    const bool swz_kind = gather || (kind == JIT_BULK && !bcast && p.k <= 16);
    const bool k128 = (p.k * (int)sizeof(T)) % 128 == 0;
    const bool asw_ok = swz_kind && !devab && opa != OP_N && k128;
    const bool bsw_ok = swz_kind && !devab && opb == OP_N && k128;
    // FP64 tensor cores (mma_item, one warp per macro-tile) for d / z
    const int mmode = mma_mode();
    const bool mma = MmaOk<T>::value && !devab && !bcast &&
                     (mmode == 1 || (mmode < 0 && mma_jit_rule(cplx, p.m, p.n, p.k,
                                                               kind != JIT_BULK && kind != JIT_GATHER)));
    JitMap mp = jit_mapping((int)sizeof(T), cplx, p.m, p.n, p.k, opa, opb, b0,
                            kind != JIT_BULK, asw_ok && !mma, bsw_ok && !mma);
    if (mma) mp.ASW = mp.BSW = 0;  // the micro-tile mapping is unused
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
        if (mma) expr += ", true";
    }
    // bulk_ptr_kernel<..., MMA, DEC>: the decoupled ring for 8- and 16-byte types with a
    // C input (pointer-array A/B, round 2, profiles/r02s3_ptr_ab_dec.jsonl: d16 general
    // 0.58 -> 0.85 of HBM; it lost on beta = 0 and on s: c16 beta = 0 0.72 -> 0.57)
    const bool dec = kind == JIT_BULK_PTR && !b0 && sizeof(T) >= 8;
    if (kind == JIT_BULK_PTR) expr += std::string(mma ? ", true" : ", false") + (dec ? ", true" : ", false");
    const bool swz = kind == JIT_BULK && (mp.ASW || mp.BSW);
    if (kind == JIT_BULK && (bcast || devab || swz || mma)) {  // <..., BCAST, TRA, DEVAB, ASW, BSW[, MMA]>
        expr += ", " + std::to_string(bcast) + ", false";
        expr += devab ? ", true" : ", false";
        expr += mp.ASW ? ", true" : ", false";
        expr += mp.BSW ? ", true" : ", false";
        if (mma) expr += ", true";
    }
    expr += ">";
    CUfunction f = jit_function(expr);
    if (!f) return cudaErrorNotSupported;
    const int rows_cap = swz ? 256 / std::max(mp.ASW ? p.m : 1, mp.BSW ? p.n : 1) : 0;
    static const int gather_kb = [] {  // TX_GATHER_KB: stage-size target of the gather ring (tuning)
        const char *v = getenv("TX_GATHER_KB");
        return v ? atoi(v) : 0;
    }();
    // bulk_ptr: two stages of ~16 KB (pointer-array A/B over S x KB, round 2: s16 general
    // 0.54 -> 0.95, z16 beta = 0 0.38 -> 0.85 of HBM against the strided instance's plan)
    // strided sizes beyond 16 with a C input: two 32 KB stages (pipeline sweep, round 2,
    // profiles/r02s3_tune_big.jsonl: s40 general 0.70 -> 0.89, c17 0.65 -> 0.91, c24 0.67 ->
    // 0.87 of HBM, s24 / s48 / s56 / c28 unchanged within 0.02, s32 0.98 -> 0.96)
    const bool big_gen = kind == JIT_BULK && !b0 && !bcast && std::max(p.m, std::max(p.n, p.k)) > 16;
    // Square sizes beyond 16: two-stage plans where a pipeline sweep measured them > 3 % faster
    // than the rule above (stage KB per (type, n, beta = 0); 0 = keep).  s beta = 0:
    // profiles/r02s3_sizes17_32.jsonl (17 0.48 -> 0.73, 21 0.57 -> 0.80, 25 0.44 -> 0.66, 30 0.79
    // -> 0.93 of HBM); d / c / z: profiles/r02s3_big_tuning_cdz.jsonl (d19 general 0.84 -> 0.97,
    // d24 beta = 0 0.86 -> 0.92, c20 general 0.81 -> 0.95, c18 beta = 0 0.81 -> 0.89, z17 beta = 0
    // 0.74 -> 0.81, z20 beta = 0 0.62 -> 0.68).
    auto big_kb = [](int es, bool cplx, int n, bool beta0) -> int {
        if (n < 17 || n > 32) return 0;
        if (es == 4) return (beta0 && (n == 17 || n == 21 || n == 22 || n == 23 || n == 25 ||
                                   n == 26 || n == 30)) ? 16 : 0;
        if (es == 8 && !cplx) {  // d
            if (beta0) return (n == 17 || n == 18 || n == 20 || n == 22) ? 32
                          : (n == 19 || n == 21 || n == 23 || n == 24 || n == 27 || n == 28) ? 64 : 0;
            return (n == 19 || n == 22 || n == 24) ? 64 : 0;
        }
        if (es == 8) return beta0 ? (n == 18 ? 16 : 0) : (n == 20 ? 64 : 0);  // c
        if (beta0) return n <= 22 ? 32 : n <= 25 ? 64 : 0;                     // z
        return (n == 20 || n == 24) ? 64 : 0;
    };
    const int sq_kb = kind == JIT_BULK && !bcast && p.m == p.n && p.n == p.k
                          ? big_kb((int)sizeof(T), cplx, p.n, b0) : 0;
    const int kb = gather && gather_kb > 0 ? gather_kb
                   : (kind == JIT_BULK_PTR ? 16 : sq_kb > 0 ? sq_kb : big_gen ? 32 : mp.KB);
    static const bool two_ctas = [] {  // TX_PLAN_2CTA=0: the plain planner (A/B runs)
        const char *v = getenv("TX_PLAN_2CTA");
        return !(v && v[0] == '0');
    }();
    Plan pl = plan_tiles(sizeof(T), p.m, p.n, p.k, b0, mp.RM, mp.RN, NT, p.batch, !gather,
                         gather ? GS : (kind == JIT_BULK_PTR || big_gen || sq_kb > 0 ? 2 : mp.S), kb, kind == JIT_BULK ? bcast : 0, 0, rows_cap,
                         kind == JIT_BULK && two_ctas, mma ? 32 * mma_items(cplx, p.m, p.n) : 0);
    if (swz) {
        // the 1024-byte alignment of the swizzled regions: shrink the tile until it fits
        const int es = (int)sizeof(T);
        const int unit = 16 / gcd_i(16, gcd_i(p.m * p.k * es, gcd_i(p.k * p.n * es, p.m * p.n * es)));
        auto smem_of = [&](int P) {
            return swz_smem(pl.S, P, es, p.m, p.n, p.k, b0, mp.ASW != 0, mp.BSW != 0);
        };
        // fewer stages first (keeps the tile, i.e. whole passes of the thread block), then P
        while (smem_of(pl.P) > SMEM_MAX_BYTES && pl.S > 2) --pl.S;
        while (smem_of(pl.P) > SMEM_MAX_BYTES && pl.P > unit) pl.P -= unit;
        // two resident CTAs where a full pass of the thread block still fits (one CTA of
        // 4 warps leaves the copies' latency exposed: ncu, z 16x3x16 TT)
        const int tpm = ((p.m + mp.RM - 1) / mp.RM) * ((p.n + mp.RN - 1) / mp.RN);
        const int ppass = std::max(1, NT / tpm);
        while (smem_of(pl.P) > SMEM_BUDGET_BYTES) {
            if (pl.P - unit >= ppass) pl.P -= unit;
            else if (pl.S > 2) --pl.S;
            else break;
        }
        pl.smem = smem_of(pl.P);
        pl.ntiles = (int)(((long long)p.batch + pl.P - 1) / pl.P);
        if (pl.smem > SMEM_MAX_BYTES) return cudaErrorNotSupported;
        if (mp.ASW && !encode_tma_rows(&p.tma_a, p.A, (int)sizeof(T), p.k,
                                       (long long)p.batch * p.m, pl.P * p.m))
            return cudaErrorNotSupported;
        if (mp.BSW && !encode_tma_rows(&p.tma_b, p.B, (int)sizeof(T), p.k,
                                       (long long)p.batch * p.n, pl.P * p.n))
            return cudaErrorNotSupported;
    }
    if (kind == JIT_GATHER_PTR || kind == JIT_GATHER_PTR16)
        gather_ptr_plan(pl, (int)sizeof(T), p.m, p.n, p.k, b0, p.batch);
    if (kind == JIT_BULK_PTR && pl.P > 128) {  // bulk_ptr_kernel: <= 4 pointer triples per lane
        pl.P = 128;
        pl.ntiles = (int)(((long long)p.batch + 127) / 128);
        const int SA = p.m * p.k, SB = p.k * p.n, SC = p.m * p.n;
        pl.smem = pl.S * 128 * (SA + SB + (b0 ? 0 : SC)) * (int)sizeof(T) + 16 * pl.S;  // full + empty barriers
    }
    if (kind == JIT_BULK_PTR) pl.smem += pl.S * pl.P * 8;  // the C-pointer slots
    if (pl.smem > SMEM_MAX_BYTES) return cudaErrorNotSupported;  // the caller gathers
    p.P = pl.P;
    p.S = pl.S;
    p.ntiles = pl.ntiles;
    int occ = jit_occupancy(f, NT, pl.smem);
    if (ctas_per_sm_cap() > 0 && occ > ctas_per_sm_cap()) occ = ctas_per_sm_cap();
    long long grid = (long long)num_sms() * occ;
    const int cap = max_ctas_override();
    if (cap > 0 && grid > cap) grid = cap;
    if (grid > pl.ntiles) grid = pl.ntiles;
    if (grid < 1) grid = 1;
    return jit_launch(f, (int)grid, NT, pl.smem, st, &p);
}

}  // namespace tx
