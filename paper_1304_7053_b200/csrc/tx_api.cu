// tx_api.cu -- the C ABI (include/txgemm.h): argument validation, alpha/beta and
// layout classification, instance selection and launch.  Host code only.
//
// Call stack: tx_gemm_batched_<t> -> validate (pure host, no
// CUDA call) -> quick return | scale kernel (alpha == 0 or k == 0) | bulk kernel
// (packed, aligned; size-specialised when m == n == k) [+ gather tail] | gather
// kernel (any other strided layout) ; tx_gemm_batched_ptr_<t> -> gather kernel
// over the pointer arrays.
#include <cuda.h>  // CUtensorMap types only (the entry point is resolved at run time)

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "txgemm.h"
#include "tx_dispatch.cuh"
#include "tx_jit.h"

namespace tx {

#define TX_DECL_BULK(t, a) void register_bulk_##t##_##a(TypeTables &);
TX_DECL_BULK(0, 0)
TX_DECL_BULK(0, 1)
TX_DECL_BULK(1, 0)
TX_DECL_BULK(1, 1)
TX_DECL_BULK(2, 0)
TX_DECL_BULK(2, 1)
TX_DECL_BULK(2, 2)
TX_DECL_BULK(3, 0)
TX_DECL_BULK(3, 1)
TX_DECL_BULK(3, 2)
void register_gen_0(TypeTables &);
void register_gen_1(TypeTables &);
void register_gen_2(TypeTables &);
void register_gen_3(TypeTables &);

static TypeTables g_tab[4];
static std::once_flag g_once;

TypeTables &tables(int t)
{
    std::call_once(g_once, [] {
        std::memset(g_tab, 0, sizeof(g_tab));
        register_bulk_0_0(g_tab[0]);
        register_bulk_0_1(g_tab[0]);
        register_bulk_1_0(g_tab[1]);
        register_bulk_1_1(g_tab[1]);
        register_bulk_2_0(g_tab[2]);
        register_bulk_2_1(g_tab[2]);
        register_bulk_2_2(g_tab[2]);
        register_bulk_3_0(g_tab[3]);
        register_bulk_3_1(g_tab[3]);
        register_bulk_3_2(g_tab[3]);
        register_gen_0(g_tab[0]);
        register_gen_1(g_tab[1]);
        register_gen_2(g_tab[2]);
        register_gen_3(g_tab[3]);
    });
    return g_tab[t];
}

static std::atomic<int> g_max_ctas{0};
int max_ctas_override() { return g_max_ctas.load(std::memory_order_relaxed); }
// TX_CTAS_PER_SM: cap on resident CTAs per SM for the persistent grids (A/B measurements)
int ctas_per_sm_cap()
{
    static const int v = [] {
        const char *e = getenv("TX_CTAS_PER_SM");
        return e && *e ? atoi(e) : 0;
    }();
    return v;
}
static std::atomic<int> g_tune_stages{0}, g_tune_kb{0};
int tune_stages() { return g_tune_stages.load(std::memory_order_relaxed); }
int tune_stage_bytes() { return g_tune_kb.load(std::memory_order_relaxed) * 1024; }

int num_sms()
{
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 1;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

static thread_local int t_last_path = 0;
static thread_local int t_last_launches = 0;
static thread_local bool t_prepare = false;
bool prepare_only() { return t_prepare; }

// ---------------------------------------------------------------- scalars
template <class U> struct Api;
template <> struct Api<float> {
    using T = float;
    static constexpr int id = 0;
    static constexpr bool cplx = false;
    static bool zero(const float &v) { return v == 0.f; }
    static bool one(const float &v) { return v == 1.f; }
    static T dev(const float &v) { return v; }
};
template <> struct Api<double> {
    using T = double;
    static constexpr int id = 1;
    static constexpr bool cplx = false;
    static bool zero(const double &v) { return v == 0.0; }
    static bool one(const double &v) { return v == 1.0; }
    static T dev(const double &v) { return v; }
};
template <> struct Api<tx_cfloat> {
    using T = float2;
    static constexpr int id = 2;
    static constexpr bool cplx = true;
    static bool zero(const tx_cfloat &v) { return v.re == 0.f && v.im == 0.f; }
    static bool one(const tx_cfloat &v) { return v.re == 1.f && v.im == 0.f; }
    static T dev(const tx_cfloat &v) { return make_float2(v.re, v.im); }
};
template <> struct Api<tx_cdouble> {
    using T = double2;
    static constexpr int id = 3;
    static constexpr bool cplx = true;
    static bool zero(const tx_cdouble &v) { return v.re == 0.0 && v.im == 0.0; }
    static bool one(const tx_cdouble &v) { return v.re == 1.0 && v.im == 0.0; }
    static T dev(const tx_cdouble &v) { return make_double2(v.re, v.im); }
};
static_assert(sizeof(tx_cfloat) == sizeof(float2), "layout");
static_assert(TX_MAX_DIM == TXK_MAX_DIM, "size limit");
static_assert(sizeof(tx_cdouble) == sizeof(double2), "layout");

// ------------------------------------------------------------- validation
static bool op_ok(char c) { return c == 'n' || c == 'N' || c == 't' || c == 'T' || c == 'c' || c == 'C'; }
static bool op_n(char c) { return c == 'n' || c == 'N'; }
static int op_code(char c, bool cplx)
{
    if (op_n(c)) return OP_N;
    if ((c == 'c' || c == 'C') && cplx) return OP_C;
    return OP_T;  // 'C' on a real type is 'T' (reading R6)
}
static int max1(int v) { return v > 1 ? v : 1; }

static long long extent_elems(int rows, int cols, int ld, long long ld2, int batch)
{
    if (rows <= 0 || cols <= 0 || batch <= 0) return 0;
    return ld2 * (long long)(batch - 1) + (long long)ld * (cols - 1) + rows;
}

static bool overlap(const void *p, long long np, const void *q, long long nq, size_t es)
{
    if (np <= 0 || nq <= 0) return false;
    const uintptr_t a0 = (uintptr_t)p, a1 = a0 + (uintptr_t)np * es;
    const uintptr_t b0 = (uintptr_t)q, b1 = b0 + (uintptr_t)nq * es;
    return a0 < b1 && b0 < a1;
}

// Checks in the order documented in include/txgemm.h.  ptr = pointer-array call.
static int validate(bool ptr, char ta, char tb, int m, int n, int k, const void *alpha,
                    bool alpha_zero, const void *beta, const void *A, int lda, long long lda2,
                    const void *B, int ldb, long long ldb2, const void *C, int ldc,
                    long long ldc2, int batch, size_t es, bool cplx)
{
    const int maxdim = cplx ? TX_MAX_DIM_CPLX : TX_MAX_DIM;
    if (!op_ok(ta)) return -1;
    if (!op_ok(tb)) return -2;
    if (m < 0 || m > maxdim) return -3;
    if (n < 0 || n > maxdim) return -4;
    if (k < 0 || k > maxdim) return -5;
    if (!alpha) return -6;
    if (!beta) return ptr ? -11 : -13;
    const int rowsA = op_n(ta) ? m : k, colsA = op_n(ta) ? k : m;
    const int rowsB = op_n(tb) ? k : n, colsB = op_n(tb) ? n : k;
    if (lda < max1(rowsA)) return -8;
    if (ldb < max1(rowsB)) return ptr ? -10 : -11;
    if (ldc < max1(m)) return ptr ? -13 : -15;
    if (!ptr && batch > 1) {
        if (lda2 < 0) return -9;
        if (ldb2 < 0) return -12;
        if (ldc2 < (long long)ldc * n) return -16;
    }
    if (batch < 0) return ptr ? -14 : -17;
    const bool work = m > 0 && n > 0 && batch > 0;
    const bool reads_ab = work && !alpha_zero && k > 0;
    // NULL, or not aligned to the element size (s 4, d 8, c 8, z 16 bytes: the
    // kernels move whole elements / element pairs); the pointer arrays themselves
    // must be aligned to 8 bytes
    const size_t al = ptr ? sizeof(void *) : es;
    auto bad = [al](const void *q) { return !q || ((uintptr_t)q % al) != 0; };
    if (reads_ab && bad(A)) return -7;
    if (reads_ab && bad(B)) return ptr ? -9 : -10;
    if (work && bad(C)) return ptr ? -12 : -14;
    if (!ptr && reads_ab) {
        const long long ec = extent_elems(m, n, ldc, ldc2, batch);
        if (overlap(C, ec, A, extent_elems(rowsA, colsA, lda, lda2, batch), es)) return -14;
        if (overlap(C, ec, B, extent_elems(rowsB, colsB, ldb, ldb2, batch), es)) return -14;
    }
    return 0;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// ASW tensor map (tx_dispatch.cuh): stored A viewed as `rows` rows of k*es bytes
// in 8-byte units; rows longer than 128 B are a 3-D view {16 units, regions,
// rows} so each box covers one 128-byte region of box_rows rows.  128-byte
// swizzle, zero fill past the last row.  cuTensorMapEncodeTiled is resolved
// through cudaGetDriverEntryPoint (no link-time libcuda dependency).
bool encode_tma_rows(TmaDesc *d, const void *base, int es, int k, long long rows, int box_rows)
{
    using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn enc = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeFn) nullptr;
        return (EncodeFn)f;
    }();
    const int row_bytes = k * es;
    if (!enc || row_bytes % 128 || box_rows < 1 || box_rows > 256 || rows < 1) return false;
    static_assert(sizeof(CUtensorMap) == sizeof(TmaDesc), "tensor map size");
    const cuuint32_t regions = (cuuint32_t)(row_bytes / 128);
    CUtensorMap map;
    CUresult r;
    const cuuint32_t estr[3] = {1, 1, 1};
    if (regions == 1) {
        const cuuint64_t dims[2] = {16, (cuuint64_t)rows};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(base), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const cuuint64_t dims[3] = {16, regions, (cuuint64_t)rows};
        const cuuint64_t strides[2] = {128, (cuuint64_t)row_bytes};
        const cuuint32_t box[3] = {16, 1, (cuuint32_t)box_rows};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void *>(base), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(d, &map, sizeof(map));
    return true;
}

static int as_status(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

// FP64 tensor-core (DMMA) instances for d / z: TX_DMMA=0 never, =1 always (A/B
// measurements); unset: square AOT instances per tx_mma_table.inc, runtime-
// specialised shapes by mma_jit_rule.
int mma_mode()
{
    static const int mode = [] {
        const char *v = getenv("TX_DMMA");
        if (!v || !*v) return -1;
        return v[0] == '0' ? 0 : 1;
    }();
    return mode;
}

// Runtime-specialised shapes (non-square, pointer arrays, padded layouts): the
// tensor-core instance where measured faster (DMMA).
bool mma_jit_rule(bool cplx, int m, int n, int k, bool ptr)
{
    // pointer arrays with m or n below one 8 x 8 fragment: mostly padding (ptr A/B, round 2:
    // z 1x16x16 0.69 -> 0.91 of HBM and z 16x3x16 0.56 -> 0.92 without, profiles/r02s3_ptr_ab)
    if (ptr && std::min(m, n) < 8) return false;
    const int mx = std::max(m, std::max(n, k));
    // sizes beyond 16 (DMMA on/off sweep, round 2, profiles/r02s3_big_dmma_ab.jsonl): the
    // CUDA-core kernel wins for z 17-24 (z17 0.37-0.48 -> 0.78-0.93 of HBM, z20 0.46-0.57 ->
    // 0.64-0.77, z24 beta = 0 0.59 -> 0.80) and d 33-47 (d40 0.49-0.63 -> 0.75-0.92); DMMA
    // for z28-32 (0.64-0.85 vs 0.43-0.60) and d17-32 / d48-64
    if (cplx) return mx >= 13 && (mx <= 16 || mx >= 26);
    return mx >= 17 && !(mx >= 33 && mx <= 47);
}

// tcgen05 split-TF32 kernel for s / c (TX_TC=0 never, =1 wherever it applies:
// A/B measurements); unset: tc_rule, the sizes where the FP32 FMA pipe bounds the
// CUDA-core kernels (tensor cores).
static std::atomic<int> g_tc_override{-2};  // tx_set_tc; -2 = not set (environment)

int tc_mode()
{
    const int o = g_tc_override.load();
    if (o >= -1) return o;
    static const int mode = [] {
        const char *v = getenv("TX_TC");
        if (!v || !*v) return -1;
        return v[0] == '0' ? 0 : 1;
    }();
    return mode;
}

bool tc_rule(bool cplx, int m, int n, int k)
{
    // From the interleaved A/B of the gate protocol (TX_TC=1 vs 0, squares 17-64 for s and
    // 9-32 for c, N/N and T/T (c: N/N, C/T, T/C), both epilogues): the
    // tensor-core kernel wins for s at 57 and above, and from 43 where a matrix's element
    // count is not a multiple of 4 (the CUDA-core bulk path then needs 4-pair tiles and
    // degrades), and for c from 29.
    const int mx = std::max(m, std::max(n, k));
    if (cplx) return mx >= 29;
    const bool odd = ((m * k) | (k * n) | (m * n)) & 3;
    return mx >= 57 || (mx >= 43 && odd);
}

// The kernel applies to packed s / c batches with m, n, k <= 64 (s) / 32 (c).
static bool tc_applies(bool cplx, int m, int n, int k)
{
    const int lim = cplx ? 32 : 64;
    if (m > lim || n > lim || k > lim) return false;
    const int mode = tc_mode();
    return mode == 1 || (mode < 0 && tc_rule(cplx, m, n, k));
}

// Register-direct kernel for n <= 2 (TX_DIRECT=0 disables it: A/B measurements).
static bool direct_enabled()
{
    static const bool on = [] {
        const char *v = getenv("TX_DIRECT");
        return !(v && v[0] == '0');
    }();
    return on;
}

// Smallest matrix (bytes) for which a packed pointer-array batch takes the per-matrix
// bulk-copy kernel instead of the 16-byte gather (TX_PTR_BULK_MIN: A/B measurements).
static int ptr_bulk_min_bytes()
{
    static const int v = [] {
        const char *e = getenv("TX_PTR_BULK_MIN");
        return e && *e ? atoi(e) : 512;
    }();
    return v;
}

// Pairs per bulk launch (a multiple of every 16-byte alignment unit): keeps the
// 32-bit TMA row coordinates pair * rows (rows <= 32) below 2^31.
constexpr long long BULK_CHUNK_PAIRS = 1ll << 26;

// ------------------------------------------------------------- strided call
template <class U>
static int gemm_strided(char ta, char tb, int m, int n, int k, const U *alpha, const U *A, int lda,
                        long long lda2, const U *B, int ldb, long long ldb2, const U *beta, U *C,
                        int ldc, long long ldc2, int batch, cudaStream_t st)
{
    using AT = Api<U>;
    using T = typename AT::T;
    const int rc = validate(false, ta, tb, m, n, k, alpha, alpha && AT::zero(*alpha), beta, A, lda,
                            lda2, B, ldb, ldb2, C, ldc, ldc2, batch, sizeof(U), AT::cplx);
    if (rc) return rc;
    const U a = *alpha, b = *beta;
    if (m == 0 || n == 0 || batch == 0 || ((AT::zero(a) || k == 0) && AT::one(b))) {
        t_last_path = PATH_NONE;
        t_last_launches = 0;
        return 0;
    }
    TypeTables &tab = tables(AT::id);
    const bool b0 = AT::zero(b);
    Params<T> p;
    std::memset(&p, 0, sizeof(p));
    p.A = reinterpret_cast<const T *>(A);
    p.B = reinterpret_cast<const T *>(B);
    p.C = reinterpret_cast<T *>(C);
    p.lda = lda;
    p.ldb = ldb;
    p.ldc = ldc;
    p.lda2 = lda2;
    p.ldb2 = ldb2;
    p.ldc2 = ldc2;
    p.m = m;
    p.n = n;
    p.k = k;
    p.batch = batch;
    p.alpha = AT::dev(a);
    p.beta = AT::dev(b);

    if (AT::zero(a) || k == 0) {
        const cudaError_t e = tab.scale[0][b0](&p, st);
        if (e != cudaSuccess) return as_status(e);
        t_last_path = PATH_SCALE;
        t_last_launches = 1;
        return 0;
    }
    const int opa = op_code(ta, AT::cplx), opb = op_code(tb, AT::cplx);
    const int rowsA = op_n(ta) ? m : k, colsA = op_n(ta) ? k : m;
    const int rowsB = op_n(tb) ? k : n, colsB = op_n(tb) ? n : k;
    const long long SA = (long long)rowsA * colsA, SB = (long long)rowsB * colsB,
                    SC = (long long)m * n;
    const bool one = batch == 1;
    const bool packed = lda == rowsA && ldb == rowsB && ldc == m &&
                        (one || (lda2 == SA && ldb2 == SB && ldc2 == SC)) && aligned16(A) &&
                        aligned16(B) && aligned16(C);
    int path = PATH_GATHER, launches = 0;
    // tensor-core kernel (s / c beyond 16): packed leading dimensions, any element
    // alignment (it copies 16-byte-aligned windows), the whole batch in one launch
    const bool packed_ld = lda == rowsA && ldb == rowsB && ldc == m &&
                           (one || (lda2 == SA && ldb2 == SB && ldc2 == SC));
    if (packed_ld && tab.tc[opa][opb][b0] && tc_applies(AT::cplx, m, n, k)) {
        const cudaError_t e = tab.tc[opa][opb][b0](&p, st);
        if (e == cudaSuccess) {
            t_last_path = PATH_TC;
            t_last_launches = 1;
            return 0;
        }
        if (e != cudaErrorNotSupported) return as_status(e);
    }
    // fixed-operand batches (the paper's §9 variant): A and/or B shared by every pair
    const bool bcA = !one && lda2 == 0 && lda == rowsA;
    const bool bcB = !one && ldb2 == 0 && ldb == rowsB;
    const bool okA = bcA || (lda == rowsA && (one || lda2 == SA) && aligned16(A));
    const bool okB = bcB || (ldb == rowsB && (one || ldb2 == SB) && aligned16(B));
    const bool okC = ldc == m && (one || ldc2 == SC) && aligned16(C);
    if (!packed && (bcA || bcB) && okA && okB && okC && jit_available()) {
        const int es = (int)sizeof(U);
        const int bcast = (bcA ? 1 : 0) | (bcB ? 2 : 0);
        int g = (int)(SC * es);
        if (!bcA) g = gcd_i(g, (int)(SA * es));
        if (!bcB) g = gcd_i(g, (int)(SB * es));
        const int unit = 16 / gcd_i(16, g);
        const int main_pairs = batch / unit * unit;
        if (main_pairs > 0) {
            Params<T> q = p;
            q.batch = main_pairs;
            const cudaError_t e = launch_jit<T>(JIT_BULK, q, opa, opb, b0, st, bcast);
            if (e != cudaSuccess && e != cudaErrorNotSupported) return as_status(e);
            if (e == cudaSuccess) {
                ++launches;
                path = PATH_BULK | PATH_JIT;
                if (main_pairs < batch) {
                    Params<T> r = p;
                    r.batch = batch - main_pairs;
                    if (!bcA) r.A += lda2 * main_pairs;
                    if (!bcB) r.B += ldb2 * main_pairs;
                    r.C += ldc2 * main_pairs;
                    const cudaError_t e2 = tab.gather[opa][opb][b0][0](&r, st);
                    if (e2 != cudaSuccess) return as_status(e2);
                    ++launches;
                    path |= PATH_TAIL;
                }
                t_last_path = path;
                t_last_launches = launches;
                return 0;
            }
        }
    }
    if (packed && m == n && n == k && m <= 2 && direct_enabled()) {
        // tiny matrices: register-direct kernel, whole batch (tail included)
        const cudaError_t e = tab.direct[opa][opb][b0][m - 1](&p, st);
        if (e != cudaSuccess) return as_status(e);
        t_last_path = PATH_DIRECT;
        t_last_launches = 1;
        return 0;
    }
    if (packed) {
        const int es = (int)sizeof(U);
        const int unit = 16 / gcd_i(16, gcd_i((int)(SA * es), gcd_i((int)(SB * es), (int)(SC * es))));
        const int main_pairs = batch / unit * unit;
        // Launches of at most BULK_CHUNK_PAIRS pairs: the TMA tensor-copy
        // coordinates (row = pair * rows, 32-bit) stay below 2^31 for rows <= 32.
        for (long long c0 = 0; c0 < main_pairs; c0 += BULK_CHUNK_PAIRS) {
            Params<T> q = p;
            q.batch = (int)std::min<long long>(BULK_CHUNK_PAIRS, main_pairs - c0);
            q.lda2 = SA;
            q.ldb2 = SB;
            q.ldc2 = SC;
            q.A += SA * c0;
            q.B += SB * c0;
            q.C += SC * c0;
            LaunchFn fn = nullptr;
            if (m == n && n == k && m <= 16) {
                fn = tab.bulk_sq[opa][opb][b0][m - 1];
                const int mode = mma_mode();
                if (tab.bulk_mma[opa][opb][b0][m - 1] &&
                    (mode == 1 || (mode < 0 && tab.mma_on[opa][opb][b0][m - 1])))
                    fn = tab.bulk_mma[opa][opb][b0][m - 1];
            }
            cudaError_t e = cudaErrorNotSupported;
            path = PATH_BULK;
            if (!fn) {  // no AOT instance for this shape: runtime-specialised instance
                e = launch_jit<T>(JIT_BULK, q, opa, opb, b0, st);
                if (e == cudaSuccess) path |= PATH_JIT;
            }
            if (e == cudaErrorNotSupported && fn) e = fn(&q, st);
            // (an AOT tensor-copy instance whose tensor map cannot be encoded also
            // reports cudaErrorNotSupported: the generic bulk kernel takes over)
            if (e == cudaErrorNotSupported) e = tab.bulk_dyn[opa][opb][b0](&q, st);
            // two stages of one alignment unit of pairs exceed shared memory (odd sizes
            // beyond ~48): the gather kernels, which need no alignment unit
            if (e == cudaErrorNotSupported) {
                e = launch_jit<T>(JIT_GATHER, q, opa, opb, b0, st);
                if (e == cudaSuccess) path = PATH_GATHER | PATH_JIT;
                if (e == cudaErrorNotSupported) {
                    e = tab.gather[opa][opb][b0][0](&q, st);
                    path = PATH_GATHER;
                }
            }
            if (e != cudaSuccess) return as_status(e);
            ++launches;
        }
        if (main_pairs < batch) {  // < 16 trailing pairs whose bytes are not 16-aligned
            Params<T> q = p;
            q.batch = batch - main_pairs;
            q.lda2 = SA;
            q.ldb2 = SB;
            q.ldc2 = SC;
            q.A += SA * main_pairs;
            q.B += SB * main_pairs;
            q.C += SC * main_pairs;
            const cudaError_t e = tab.gather[opa][opb][b0][0](&q, st);
            if (e != cudaSuccess) return as_status(e);
            ++launches;
            path = main_pairs > 0 ? (path | PATH_TAIL) : PATH_GATHER;
        }
    } else {
        cudaError_t e = launch_jit<T>(JIT_GATHER, p, opa, opb, b0, st);
        if (e == cudaSuccess) path |= PATH_JIT;
        if (e == cudaErrorNotSupported) e = tab.gather[opa][opb][b0][0](&p, st);
        if (e != cudaSuccess) return as_status(e);
        launches = 1;
    }
    t_last_path = path;
    t_last_launches = launches;
    return 0;
}

// ------------------------------------------- device-resident alpha / beta
// The values are only known on the device: the kernels decide alpha == 0 and
// beta == 0 at run time (R12).  A and B must be valid whenever
// m*n*batch > 0 and k > 0 (they may be read).
template <class U>
static int gemm_strided_dev(char ta, char tb, int m, int n, int k, const U *alpha, const U *A,
                            int lda, long long lda2, const U *B, int ldb, long long ldb2,
                            const U *beta, U *C, int ldc, long long ldc2, int batch,
                            cudaStream_t st)
{
    using AT = Api<U>;
    using T = typename AT::T;
    const int rc = validate(false, ta, tb, m, n, k, alpha, false, beta, A, lda, lda2, B, ldb,
                            ldb2, C, ldc, ldc2, batch, sizeof(U), AT::cplx);
    if (rc) return rc;
    if (m == 0 || n == 0 || batch == 0) {
        t_last_path = PATH_NONE;
        t_last_launches = 0;
        return 0;
    }
    TypeTables &tab = tables(AT::id);
    Params<T> p;
    std::memset(&p, 0, sizeof(p));
    p.A = reinterpret_cast<const T *>(A);
    p.B = reinterpret_cast<const T *>(B);
    p.C = reinterpret_cast<T *>(C);
    p.lda = lda;
    p.ldb = ldb;
    p.ldc = ldc;
    p.lda2 = lda2;
    p.ldb2 = ldb2;
    p.ldc2 = ldc2;
    p.m = m;
    p.n = n;
    p.k = k;
    p.batch = batch;
    p.alpha_dev = reinterpret_cast<const T *>(alpha);
    p.beta_dev = reinterpret_cast<const T *>(beta);
    cudaError_t e;
    if (k == 0) {
        e = tab.scale_dev[0](&p, st);
        if (e != cudaSuccess) return as_status(e);
        t_last_path = PATH_SCALE;
        t_last_launches = 1;
        return 0;
    }
    const int opa = op_code(ta, AT::cplx), opb = op_code(tb, AT::cplx);
    const int rowsA = op_n(ta) ? m : k, colsA = op_n(ta) ? k : m;
    const int rowsB = op_n(tb) ? k : n, colsB = op_n(tb) ? n : k;
    const long long SA = (long long)rowsA * colsA, SB = (long long)rowsB * colsB,
                    SC = (long long)m * n;
    const bool one = batch == 1;
    const bool packed = lda == rowsA && ldb == rowsB && ldc == m &&
                        (one || (lda2 == SA && ldb2 == SB && ldc2 == SC)) && aligned16(A) &&
                        aligned16(B) && aligned16(C);
    int launches = 0, path = PATH_GATHER;
    if (packed) {
        const int es = (int)sizeof(U);
        const int unit = 16 / gcd_i(16, gcd_i((int)(SA * es), gcd_i((int)(SB * es), (int)(SC * es))));
        const int main_pairs = batch / unit * unit;
        if (main_pairs > 0) {
            Params<T> q = p;
            q.batch = main_pairs;
            q.lda2 = SA;
            q.ldb2 = SB;
            q.ldc2 = SC;
            e = launch_jit<T>(JIT_BULK, q, opa, opb, false, st, 0, true);
            path = PATH_BULK | (e == cudaSuccess ? PATH_JIT : 0);
            if (e == cudaErrorNotSupported) e = tab.bulk_dyn_dev[opa][opb](&q, st);
            if (e == cudaErrorNotSupported) {  // does not fit (see gemm_strided): gather
                e = tab.gather_dev[opa][opb][0](&q, st);
                path = PATH_GATHER;
            }
            if (e != cudaSuccess) return as_status(e);
            ++launches;
        }
        if (main_pairs < batch) {
            Params<T> q = p;
            q.batch = batch - main_pairs;
            q.lda2 = SA;
            q.ldb2 = SB;
            q.ldc2 = SC;
            q.A += SA * main_pairs;
            q.B += SB * main_pairs;
            q.C += SC * main_pairs;
            e = tab.gather_dev[opa][opb][0](&q, st);
            if (e != cudaSuccess) return as_status(e);
            ++launches;
            path = main_pairs > 0 ? (path | PATH_TAIL) : PATH_GATHER;
        }
    } else {
        e = launch_jit<T>(JIT_GATHER, p, opa, opb, false, st, 0, true);
        if (e == cudaSuccess) path |= PATH_JIT;
        if (e == cudaErrorNotSupported) e = tab.gather_dev[opa][opb][0](&p, st);
        if (e != cudaSuccess) return as_status(e);
        launches = 1;
    }
    t_last_path = path;
    t_last_launches = launches;
    return 0;
}

template <class U>
static int gemm_ptr_dev(char ta, char tb, int m, int n, int k, const U *alpha, const U *const *Aa,
                        int lda, const U *const *Ba, int ldb, const U *beta, U *const *Ca, int ldc,
                        int batch, cudaStream_t st)
{
    using AT = Api<U>;
    using T = typename AT::T;
    const int rc = validate(true, ta, tb, m, n, k, alpha, false, beta, Aa, lda, 0, Ba, ldb, 0, Ca,
                            ldc, 0, batch, sizeof(U), AT::cplx);
    if (rc) return rc;
    if (m == 0 || n == 0 || batch == 0) {
        t_last_path = PATH_NONE;
        t_last_launches = 0;
        return 0;
    }
    TypeTables &tab = tables(AT::id);
    Params<T> p;
    std::memset(&p, 0, sizeof(p));
    p.Ap = reinterpret_cast<const T *const *>(Aa);
    p.Bp = reinterpret_cast<const T *const *>(Ba);
    p.Cp = reinterpret_cast<T *const *>(Ca);
    p.lda = lda;
    p.ldb = ldb;
    p.ldc = ldc;
    p.m = m;
    p.n = n;
    p.k = k;
    p.batch = batch;
    p.alpha_dev = reinterpret_cast<const T *>(alpha);
    p.beta_dev = reinterpret_cast<const T *>(beta);
    cudaError_t e;
    if (k == 0) {
        e = tab.scale_dev[1](&p, st);
        t_last_path = PATH_SCALE;
    } else {
        const int opa = op_code(ta, AT::cplx), opb = op_code(tb, AT::cplx);
        const int rowsA = op_n(ta) ? m : k, rowsB = op_n(tb) ? k : n;
        const int es = (int)sizeof(U);
        const bool v16 = lda == rowsA && ldb == rowsB && ldc == m && (m * k * es) % 16 == 0 &&
                         (k * n * es) % 16 == 0 && (m * n * es) % 16 == 0;
        e = launch_jit<T>(v16 ? JIT_GATHER_PTR16 : JIT_GATHER_PTR, p, opa, opb, false, st, 0, true);
        t_last_path = PATH_PTR | (e == cudaSuccess ? PATH_JIT : 0);
        if (e == cudaErrorNotSupported) e = tab.gather_dev[opa][opb][1](&p, st);
    }
    if (e != cudaSuccess) return as_status(e);
    t_last_launches = 1;
    return 0;
}

// -------------------------------------------------------- pointer-array call
template <class U>
static int gemm_ptr(char ta, char tb, int m, int n, int k, const U *alpha, const U *const *Aa,
                    int lda, const U *const *Ba, int ldb, const U *beta, U *const *Ca, int ldc,
                    int batch, cudaStream_t st)
{
    using AT = Api<U>;
    using T = typename AT::T;
    const int rc = validate(true, ta, tb, m, n, k, alpha, alpha && AT::zero(*alpha), beta, Aa, lda,
                            0, Ba, ldb, 0, Ca, ldc, 0, batch, sizeof(U), AT::cplx);
    if (rc) return rc;
    const U a = *alpha, b = *beta;
    if (m == 0 || n == 0 || batch == 0 || ((AT::zero(a) || k == 0) && AT::one(b))) {
        t_last_path = PATH_NONE;
        t_last_launches = 0;
        return 0;
    }
    TypeTables &tab = tables(AT::id);
    const bool b0 = AT::zero(b);
    Params<T> p;
    std::memset(&p, 0, sizeof(p));
    p.Ap = reinterpret_cast<const T *const *>(Aa);
    p.Bp = reinterpret_cast<const T *const *>(Ba);
    p.Cp = reinterpret_cast<T *const *>(Ca);
    p.lda = lda;
    p.ldb = ldb;
    p.ldc = ldc;
    p.m = m;
    p.n = n;
    p.k = k;
    p.batch = batch;
    p.alpha = AT::dev(a);
    p.beta = AT::dev(b);
    cudaError_t e;
    if (AT::zero(a) || k == 0) {
        e = tab.scale[1][b0](&p, st);
        t_last_path = PATH_SCALE;
    } else {
        const int opa = op_code(ta, AT::cplx), opb = op_code(tb, AT::cplx);
        const int rowsA = op_n(ta) ? m : k, rowsB = op_n(tb) ? k : n;
        const int es = (int)sizeof(U);
        // packed matrices whose byte sizes are multiples of 16: per-matrix bulk copies
        const bool bulk_ok = lda == rowsA && ldb == rowsB && ldc == m && (m * k * es) % 16 == 0 &&
                             (k * n * es) % 16 == 0 && (m * n * es) % 16 == 0;
        // small matrices: 16-byte cp.async chunks over all threads (a per-matrix
        // TMA copy costs ~80 cycles of issue); >= 512-byte matrices: TMA per matrix
        const int min_bytes = es * std::min(m * k, std::min(k * n, m * n));
        // ... except where the 16-byte gather measured faster on large matrices
        // (profiles/r02s3_ptr_ab_transA.jsonl): a transposed A without the FP64 tensor cores
        // (the gather places it swizzled, ASWG; bulk_ptr reads it with bank conflicts):
        // z 16x3x16 T/C 0.51-0.69 -> 0.61-0.81, d 16x16x16 T/C general 0.53-0.64 -> 0.68-0.77;
        // c with a C input: 16x16x16 0.50-0.69 -> 0.68-0.80
        const bool mma = MmaOk<T>::value && (mma_mode() == 1 ||
                                             (mma_mode() < 0 && mma_jit_rule(AT::cplx, m, n, k, true)));
        const bool prefer_gather = es == 16 ? (!mma && opa != OP_N)
                                   : es == 8 && !AT::cplx ? (!b0 && opa != OP_N)
                                   : es == 8 ? !b0 : false;
        const JitKind kind = !bulk_ok ? JIT_GATHER_PTR
                             : (min_bytes >= ptr_bulk_min_bytes() && !prefer_gather ? JIT_BULK_PTR
                                                                                    : JIT_GATHER_PTR16);
        e = launch_jit<T>(kind, p, opa, opb, b0, st);
        t_last_path = PATH_PTR | (e == cudaSuccess ? PATH_JIT : 0);
        if (e == cudaErrorNotSupported) e = tab.gather[opa][opb][b0][1](&p, st);
    }
    if (e != cudaSuccess) return as_status(e);
    t_last_launches = 1;
    return 0;
}

// ---------------------------------------------------------- host-buffer call
// Auxiliary copy streams (one pair per device, created once): host->device copies
// run on one, device->host on the other, the GEMM chunks on the caller's stream,
// ordered by events, so PCIe transfers in both directions overlap each other and
// the kernels.
struct CopyStreams {
    cudaStream_t h2d = nullptr, d2h = nullptr;
};
static CopyStreams copy_streams()
{
    static std::mutex mu;
    static CopyStreams per_dev[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> g(mu);
    CopyStreams &c = per_dev[dev];
    if (!c.h2d) {
        cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking);
    }
    return c;
}

constexpr long long HOSTIO_CHUNK_MB = 64;  // pipeline chunk of the host-buffer entry (measured: 4-512 MB)

template <class U>
static int gemm_hostio(char ta, char tb, int m, int n, int k, const U *alpha, const U *hA, int lda,
                       long long lda2, const U *hB, int ldb, long long ldb2, const U *beta, U *hC,
                       int ldc, long long ldc2, int batch, cudaStream_t st, U *dA, U *dB, U *dC)
{
    using AT = Api<U>;
    int rc = validate(false, ta, tb, m, n, k, alpha, alpha && AT::zero(*alpha), beta, hA, lda,
                      lda2, hB, ldb, ldb2, hC, ldc, ldc2, batch, sizeof(U), AT::cplx);
    if (rc) return rc;
    const U a = *alpha, b = *beta;
    const bool work = m > 0 && n > 0 && batch > 0;
    const bool reads_ab = work && !AT::zero(a) && k > 0;
    auto bad = [](const void *q) { return !q || ((uintptr_t)q % sizeof(U)) != 0; };
    if (reads_ab && bad(dA)) return -19;
    if (reads_ab && bad(dB)) return -20;
    if (work && bad(dC)) return -21;
    if (!work || ((AT::zero(a) || k == 0) && AT::one(b))) {
        t_last_path = PATH_NONE;
        t_last_launches = 0;
        return 0;
    }
    const int rowsA = op_n(ta) ? m : k, colsA = op_n(ta) ? k : m;
    const int rowsB = op_n(tb) ? k : n, colsB = op_n(tb) ? n : k;
    const size_t es = sizeof(U);
    const bool read_c = !AT::zero(b);
    // Chunks of whole pairs (HOSTIO_CHUNK_MB of traffic each, TX_HOSTIO_CHUNK_MB overrides);
    // ld2 == 0 operands are copied once.
    static const long long chunk_bytes = [] {
        const char *v = getenv("TX_HOSTIO_CHUNK_MB");
        const long long mb = v ? atoll(v) : HOSTIO_CHUNK_MB;
        return (mb > 0 ? mb : HOSTIO_CHUNK_MB) << 20;
    }();
    const long long per_pair = (long long)es * ((reads_ab ? lda2 + ldb2 : 0) + ldc2 * (read_c ? 2 : 1));
    long long chunk = per_pair > 0 ? chunk_bytes / per_pair : batch;
    if (chunk < 1) chunk = 1;
    const int nchunks = (int)((batch + chunk - 1) / chunk);
    CopyStreams cs = copy_streams();
    cudaEvent_t ev0;
    cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
    cudaEventRecord(ev0, st);
    cudaStreamWaitEvent(cs.h2d, ev0, 0);
    cudaStreamWaitEvent(cs.d2h, ev0, 0);
    cudaEventDestroy(ev0);
    cudaError_t e = cudaSuccess;
    int launches = 0, path = PATH_NONE;
    for (int c = 0; c < nchunks && e == cudaSuccess; ++c) {
        const long long p0 = (long long)c * chunk;
        const int nb = (int)(batch - p0 < chunk ? batch - p0 : chunk);
        const long long oa = lda2 * p0, ob = ldb2 * p0, oc = ldc2 * p0;
        if (reads_ab) {
            if (c == 0 || lda2 != 0)
                e = cudaMemcpyAsync(dA + oa, hA + oa, extent_elems(rowsA, colsA, lda, lda2, nb) * es,
                                    cudaMemcpyHostToDevice, cs.h2d);
            if (e == cudaSuccess && (c == 0 || ldb2 != 0))
                e = cudaMemcpyAsync(dB + ob, hB + ob, extent_elems(rowsB, colsB, ldb, ldb2, nb) * es,
                                    cudaMemcpyHostToDevice, cs.h2d);
        }
        const long long ec = extent_elems(m, n, ldc, ldc2, nb);
        if (e == cudaSuccess && read_c)
            e = cudaMemcpyAsync(dC + oc, hC + oc, ec * es, cudaMemcpyHostToDevice, cs.h2d);
        cudaEvent_t ein, ek;
        cudaEventCreateWithFlags(&ein, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ek, cudaEventDisableTiming);
        cudaEventRecord(ein, cs.h2d);
        cudaStreamWaitEvent(st, ein, 0);
        if (e == cudaSuccess) {
            rc = gemm_strided<U>(ta, tb, m, n, k, alpha, dA + oa, lda, lda2, dB + ob, ldb, ldb2,
                                 beta, dC + oc, ldc, ldc2, nb, st);
            if (rc) {
                cudaEventDestroy(ein);
                cudaEventDestroy(ek);
                return rc;
            }
            launches += t_last_launches;
            path = t_last_path;
        }
        cudaEventRecord(ek, st);
        cudaStreamWaitEvent(cs.d2h, ek, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hC + oc, dC + oc, ec * es, cudaMemcpyDeviceToHost, cs.d2h);
        cudaEventDestroy(ein);
        cudaEventDestroy(ek);
    }
    // the caller's stream is ordered after the last device->host copy
    cudaEvent_t eend;
    cudaEventCreateWithFlags(&eend, cudaEventDisableTiming);
    cudaEventRecord(eend, cs.d2h);
    cudaStreamWaitEvent(st, eend, 0);
    cudaEventDestroy(eend);
    if (e != cudaSuccess) return as_status(e);
    t_last_path = path;
    t_last_launches = launches;
    return 0;
}

// ------------------------------------------------------------ tx_prepare
// Runs the dispatch of a call of this shape on placeholder (never dereferenced)
// addresses with launches suppressed: every runtime-specialised instance the
// call would use is compiled and loaded on the current device, and every AOT
// kernel's attributes are set, so a later call of this shape does no NVRTC work.
template <class U>
static int prepare(char ta, char tb, int m, int n, int k, bool b0, int layout)
{
    using AT = Api<U>;
    U one, half, zero;
    std::memset(&one, 0, sizeof(U));
    std::memset(&zero, 0, sizeof(U));
    std::memset(&half, 0, sizeof(U));
    *reinterpret_cast<typename std::conditional<AT::cplx, typename std::conditional<
        sizeof(U) == 8, float, double>::type, U>::type *>(&one) = 1;
    *reinterpret_cast<typename std::conditional<AT::cplx, typename std::conditional<
        sizeof(U) == 8, float, double>::type, U>::type *>(&half) = 0.5;
    const U *beta = b0 ? &zero : &half;
    const int batch = 1 << 20;
    const int rowsA = op_n(ta) ? m : k, colsA = op_n(ta) ? k : m;
    const int rowsB = op_n(tb) ? k : n, colsB = op_n(tb) ? n : k;
    const int pad = layout == TX_LAYOUT_STRIDED ? 1 : 0;
    const int lda = max1(rowsA) + pad, ldb = max1(rowsB) + pad, ldc = max1(m) + pad;
    const long long lda2 = (long long)lda * colsA + pad, ldb2 = (long long)ldb * colsB + pad,
                    ldc2 = (long long)ldc * n + pad;
    // disjoint, 4 KB-aligned placeholder ranges (1 TB apart)
    U *A = reinterpret_cast<U *>(uintptr_t(1) << 40), *B = reinterpret_cast<U *>(uintptr_t(2) << 40),
      *C = reinterpret_cast<U *>(uintptr_t(3) << 40);
    t_prepare = true;
    int rc;
    if (layout == TX_LAYOUT_PTR)
        rc = gemm_ptr<U>(ta, tb, m, n, k, &one, reinterpret_cast<const U *const *>(A), lda,
                         reinterpret_cast<const U *const *>(B), ldb, beta,
                         reinterpret_cast<U *const *>(C), ldc, batch, 0);
    else
        rc = gemm_strided<U>(ta, tb, m, n, k, &one, A, lda, lda2, B, ldb, ldb2, beta, C, ldc,
                             ldc2, batch, 0);
    t_prepare = false;
    t_last_path = PATH_NONE;
    t_last_launches = 0;
    // validation codes of the inner call map to tx_prepare's own positions
    if (rc == -1) return -2;
    if (rc == -2) return -3;
    if (rc == -3) return -4;
    if (rc == -4) return -5;
    if (rc == -5) return -6;
    return rc < 0 ? -8 : rc;
}

}  // namespace tx

// ====================================================================== C ABI
extern "C" int tx_prepare(char type, char transa, char transb, int m, int n, int k,
                          int beta_is_zero, int layout)
{
    if (layout != TX_LAYOUT_PACKED && layout != TX_LAYOUT_STRIDED && layout != TX_LAYOUT_PTR)
        return -8;
    switch (type) {
    case 's': case 'S': return tx::prepare<float>(transa, transb, m, n, k, beta_is_zero != 0, layout);
    case 'd': case 'D': return tx::prepare<double>(transa, transb, m, n, k, beta_is_zero != 0, layout);
    case 'c': case 'C': return tx::prepare<tx_cfloat>(transa, transb, m, n, k, beta_is_zero != 0, layout);
    case 'z': case 'Z': return tx::prepare<tx_cdouble>(transa, transb, m, n, k, beta_is_zero != 0, layout);
    default: return -1;
    }
}

using namespace tx;

#define TX_STRIDED(SUF, U)                                                                        \
    extern "C" int tx_gemm_batched_##SUF(char ta, char tb, int m, int n, int k, const U *alpha,  \
                                         const U *A, int lda, long long lda2, const U *B, int ldb, \
                                         long long ldb2, const U *beta, U *C, int ldc,            \
                                         long long ldc2, int batch, tx_stream_t stream)           \
    {                                                                                             \
        return gemm_strided<U>(ta, tb, m, n, k, alpha, A, lda, lda2, B, ldb, ldb2, beta, C, ldc,  \
                               ldc2, batch, (cudaStream_t)stream);                                \
    }                                                                                             \
    extern "C" int tx_gemm_batched_ptr_##SUF(char ta, char tb, int m, int n, int k,               \
                                             const U *alpha, const U *const *Aa, int lda,         \
                                             const U *const *Ba, int ldb, const U *beta,          \
                                             U *const *Ca, int ldc, int batch,                    \
                                             tx_stream_t stream)                                  \
    {                                                                                             \
        return gemm_ptr<U>(ta, tb, m, n, k, alpha, Aa, lda, Ba, ldb, beta, Ca, ldc, batch,        \
                           (cudaStream_t)stream);                                                 \
    }                                                                                             \
    extern "C" int tx_gemm_batched_hostio_##SUF(                                                  \
        char ta, char tb, int m, int n, int k, const U *alpha, const U *hA, int lda,             \
        long long lda2, const U *hB, int ldb, long long ldb2, const U *beta, U *hC, int ldc,     \
        long long ldc2, int batch, tx_stream_t stream, U *dA, U *dB, U *dC)                      \
    {                                                                                             \
        return gemm_hostio<U>(ta, tb, m, n, k, alpha, hA, lda, lda2, hB, ldb, ldb2, beta, hC,     \
                              ldc, ldc2, batch, (cudaStream_t)stream, dA, dB, dC);                \
    }

#define TX_DEV(SUF, U)                                                                            \
    extern "C" int tx_gemm_batched_dev_##SUF(char ta, char tb, int m, int n, int k, const U *alpha,\
                                             const U *A, int lda, long long lda2, const U *B,       \
                                             int ldb, long long ldb2, const U *beta, U *C, int ldc, \
                                             long long ldc2, int batch, tx_stream_t stream)          \
    {                                                                                             \
        return gemm_strided_dev<U>(ta, tb, m, n, k, alpha, A, lda, lda2, B, ldb, ldb2, beta, C,   \
                                   ldc, ldc2, batch, (cudaStream_t)stream);                       \
    }                                                                                             \
    extern "C" int tx_gemm_batched_ptr_dev_##SUF(char ta, char tb, int m, int n, int k,           \
                                                 const U *alpha, const U *const *Aa, int lda,     \
                                                 const U *const *Ba, int ldb, const U *beta,      \
                                                 U *const *Ca, int ldc, int batch,                \
                                                 tx_stream_t stream)                              \
    {                                                                                             \
        return gemm_ptr_dev<U>(ta, tb, m, n, k, alpha, Aa, lda, Ba, ldb, beta, Ca, ldc, batch,    \
                               (cudaStream_t)stream);                                             \
    }

TX_DEV(s, float)
TX_DEV(d, double)
TX_DEV(c, tx_cfloat)
TX_DEV(z, tx_cdouble)

TX_STRIDED(s, float)
TX_STRIDED(d, double)
TX_STRIDED(c, tx_cfloat)
TX_STRIDED(z, tx_cdouble)

extern "C" const char *tx_status_string(int status)
{
    static const char *args[] = {"ok",    "transa", "transb", "m",     "n",      "k",
                                 "alpha", "A",      "lda",    "lda2",  "B",      "ldb",
                                 "ldb2",  "beta",   "C",      "ldc",   "ldc2",   "batch_count",
                                 "stream", "dA",    "dB",     "dC"};
    static thread_local char buf[96];
    if (status == 0) return "success";
    if (status < 0 && -status < (int)(sizeof(args) / sizeof(args[0]))) {
        snprintf(buf, sizeof(buf), "invalid argument %d (%s in the strided call)", -status,
                 args[-status]);
        return buf;
    }
    if (status > 0) return cudaGetErrorString((cudaError_t)status);
    return "invalid argument";
}

extern "C" int tx_version(void) { return TX_VERSION; }

extern "C" int tx_last_path(int *launches)
{
    if (launches) *launches = t_last_launches;
    return t_last_path;
}

extern "C" int tx_set_max_ctas(int v) { return g_max_ctas.exchange(v < 0 ? 0 : v); }

extern "C" int tx_set_tuning(int stages, int stage_kb)
{
    const int prev = g_tune_stages.load();
    g_tune_stages.store(stages >= 2 && stages <= 8 ? stages : 0);
    g_tune_kb.store(stage_kb > 0 && stage_kb <= 96 ? stage_kb : 0);
    return prev;
}

extern "C" int tx_set_jit(int enable) { return jit_set_enabled(enable); }

extern "C" int tx_set_tc(int mode)
{
    const int prev = tc_mode();
    g_tc_override.store(mode < 0 ? -1 : (mode ? 1 : 0));
    return prev;
}

extern "C" int tx_jit_compiled(void) { return jit_available() ? jit_compiled_count() : -1; }

extern "C" int tx_num_instances(void)
{
    int c = 0;
    for (int t = 0; t < 4; ++t) c += tables(t).count;
    return c;
}
