// tx_dispatch.cuh -- host-side planning (tile size, stages, grid) and the typed
// launch functions that populate the per-type dispatch tables.
#pragma once

#include <mutex>
#include <unordered_map>
#include <utility>

#include "tx_kernels.cuh"

namespace tx {

using LaunchFn = cudaError_t (*)(const void *params, cudaStream_t stream);

// Per scalar type: size-specialised bulk instances for square sizes 1..16 (the
// paper's regime; "more specialized kernels of a given matrix
// size") plus generic-size bulk, gather and scale kernels.
struct TypeTables {
    LaunchFn bulk_sq[3][3][2][16];  // [opa][opb][beta0][n-1]
    LaunchFn bulk_dyn[3][3][2];     // any m, n, k <= 16
    LaunchFn gather[3][3][2][2];    // [opa][opb][beta0][ptr]
    LaunchFn scale[2][2];           // [ptr][beta0]
    int count;
};
TypeTables &tables(int type_id);  // 0 s, 1 d, 2 c, 3 z  (defined in tx_api.cu)

// ---- runtime knobs shared by all instances ----
int max_ctas_override();  // tx_set_max_ctas (0 = automatic)
int num_sms();            // current device

constexpr int NT_DEFAULT = 128;
constexpr int STAGE_TARGET_BYTES = 16384;
constexpr int SMEM_BUDGET_BYTES = 110 * 1024;  // aim for 2 CTAs per SM
constexpr int SMEM_MAX_BYTES = 227 * 1024;

inline int gcd_i(int a, int b)
{
    while (b) {
        int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Micro-tile per thread: rows x cols of C (balanced split of m into blocks of
// at most 4 -- 2 for double complex, whose accumulators are 4 registers each).
template <class T>
constexpr int rm_target() { return sizeof(T) == 16 ? 2 : 4; }
constexpr int balanced(int n, int target) { return n <= 0 ? target : (n + ((n + target - 1) / target) - 1) / ((n + target - 1) / target); }

struct Plan {
    int P, S, smem, ntiles;
};

// Tile plan: P pairs per tile (a multiple of the 16-byte alignment unit for the
// bulk path), S stages, dynamic shared memory.  P is at least one full pass of
// NT threads and targets ~16 KB of input per stage; shrunk for small batches so
// every SM gets a tile.
inline Plan plan_tiles(int es, int m, int n, int k, bool b0, int rm, int rn, int nt, int batch,
                       bool bulk, int fixed_stages)
{
    const int SA = m * k, SB = k * n, SC = m * n;
    const int tpm = ((m + rm - 1) / rm) * ((n + rn - 1) / rn);
    const int in = (SA + SB + (b0 ? 0 : SC)) * es;
    const int out = bulk ? SC * es : 0;
    const int align = bulk ? 16 / gcd_i(16, gcd_i(SA * es, gcd_i(SB * es, SC * es))) : 1;
    const int ppass = nt / tpm > 0 ? nt / tpm : 1;
    int passes = STAGE_TARGET_BYTES / (ppass * in);
    if (passes < 1) passes = 1;
    int P = ppass * passes;
    // small batches: spread over the SMs
    const int sms = num_sms();
    const long long per_sm = ((long long)batch + sms - 1) / sms;
    if (per_sm < P) P = (int)per_sm;
    P = ((P + align - 1) / align) * align;
    if (P < align) P = align;
    int S = fixed_stages;
    if (S == 0) {
        S = (SMEM_BUDGET_BYTES - 2 * P * out) / (P * in);
        if (S > 4) S = 4;
        if (S < 2) S = 2;
    }
    while (S * P * in + 2 * P * out + 8 * S > SMEM_MAX_BYTES && P > align) P -= align;
    Plan pl;
    pl.P = P;
    pl.S = S;
    pl.smem = S * P * in + 2 * P * out + 8 * S;
    pl.ntiles = (int)(((long long)batch + P - 1) / P);
    return pl;
}

// Resident CTAs per SM for (kernel, smem), cached.
inline int occupancy(const void *fn, int nt, int smem)
{
    static std::mutex mu;
    static std::unordered_map<const void *, std::unordered_map<int, int>> cache;
    std::lock_guard<std::mutex> g(mu);
    auto &c = cache[fn];
    auto it = c.find(smem);
    if (it != c.end()) return it->second;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX_BYTES);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nt, smem) != cudaSuccess || occ < 1)
        occ = 1;
    c[smem] = occ;
    return occ;
}

inline int grid_for(const void *fn, int nt, int smem, long long work_units)
{
    long long g = (long long)num_sms() * occupancy(fn, nt, smem);
    const int cap = max_ctas_override();
    if (cap > 0 && g > cap) g = cap;
    if (g > work_units) g = work_units;
    if (g < 1) g = 1;
    return (int)g;
}

template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0>
cudaError_t launch_bulk(const void *vp, cudaStream_t st)
{
    Params<T> p = *static_cast<const Params<T> *>(vp);
    constexpr int RM = balanced(MS ? MS : 16, rm_target<T>());
    constexpr int RN = balanced(NS ? NS : 16, 4);
    constexpr int NT = NT_DEFAULT;
    auto kern = &bulk_kernel<T, MS, NS, KS, OPA, OPB, B0, RM, RN, NT>;
    Plan pl = plan_tiles(sizeof(T), p.m, p.n, p.k, B0, RM, RN, NT, p.batch, true, 0);
    p.P = pl.P;
    p.S = pl.S;
    p.ntiles = pl.ntiles;
    const int grid = grid_for((const void *)kern, NT, pl.smem, pl.ntiles);
    kern<<<grid, NT, pl.smem, st>>>(p);
    return cudaGetLastError();
}

template <class T, int OPA, int OPB, bool B0, bool PTR>
cudaError_t launch_gather(const void *vp, cudaStream_t st)
{
    Params<T> p = *static_cast<const Params<T> *>(vp);
    constexpr int RM = rm_target<T>();
    constexpr int RN = 4;
    constexpr int NT = NT_DEFAULT;
    auto kern = &gather_kernel<T, OPA, OPB, B0, RM, RN, NT, PTR>;
    Plan pl = plan_tiles(sizeof(T), p.m, p.n, p.k, B0, RM, RN, NT, p.batch, false, GS);
    p.P = pl.P;
    p.S = GS;
    p.ntiles = pl.ntiles;
    const int grid = grid_for((const void *)kern, NT, pl.smem, pl.ntiles);
    kern<<<grid, NT, pl.smem, st>>>(p);
    return cudaGetLastError();
}

template <class T, bool PTR, bool B0>
cudaError_t launch_scale(const void *vp, cudaStream_t st)
{
    const Params<T> &p = *static_cast<const Params<T> *>(vp);
    const long long total = (long long)p.m * p.n * p.batch;
    long long blocks = (total + 255) / 256;
    const long long cap = (long long)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    scale_kernel<T, PTR, B0><<<(int)blocks, 256, 0, st>>>(p);
    return cudaGetLastError();
}

template <class T, int OPA, int OPB, bool B0, int... Is>
void fill_square(TypeTables &t, std::integer_sequence<int, Is...>)
{
    ((t.bulk_sq[OPA][OPB][B0][Is] = &launch_bulk<T, Is + 1, Is + 1, Is + 1, OPA, OPB, B0>), ...);
    t.count += (int)sizeof...(Is);
}

}  // namespace tx
