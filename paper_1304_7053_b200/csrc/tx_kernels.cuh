// tx_kernels.cuh -- the batched small-matrix GEMM kernels for sm_100a.
//
// One pass of the hot path (Eq. (1)) for a tile of P consecutive
// matrix triples:
//   (a3) load A^p, B^p (and C^p when beta != 0) from HBM into a shared-memory stage,
//   (a4/a5) each thread computes an RM x RN register micro-tile of one C^p with
//           op() folded into the shared-memory addressing and the FMA signs,
//   (a6) epilogue y = alpha*x (+ beta*y) -- C is never read when beta == 0,
//   (a7) store C^p to HBM.
// DESIGN.md §Kernels describes the layout, the roofline and the algorithmic bytes.
//
// Two data movers share the compute core (micro_tile):
//  * bulk_kernel   -- packed, 16-byte-aligned strided batches (the paper's basic
//    layout: minimal leading dimensions).  Each tile of each
//    operand is ONE contiguous run of bytes, so a single thread moves it with a
//    1-D bulk async copy (TMA engine, cp.async.bulk) into an S-stage ring tracked
//    by mbarriers, and C goes back with a bulk store from a double-buffered
//    output tile.  Persistent CTAs loop over tiles (the paper's "each CUDA
//    thread-block is used to process multiple matrices").
//  * gather_kernel -- any strided layout (padded ld/ld2, broadcast ld2 = 0,
//    unaligned bases) and the pointer-array layout: element-
//    granular cp.async (LDGSTS) gathers into the same packed stage layout, C is
//    written straight from registers.
#pragma once

#include "tx_common.cuh"

namespace tx {

template <class T>
struct Params {
    const T *A;
    const T *B;
    T *C;
    const T *const *Ap;  // pointer-array layout
    const T *const *Bp;
    T *const *Cp;
    long long lda2, ldb2, ldc2;
    int lda, ldb, ldc;
    int m, n, k;   // runtime sizes (used when the kernel's static size is 0)
    int batch;     // pairs handled by this launch
    int P;         // pairs per tile
    int S;         // pipeline stages (bulk kernel)
    int ntiles;    // ceil(batch / P)
    T alpha, beta;
};

// --------------------------------------------------------------------------
// Register micro-tile: rows i0..i0+RM-1, cols j0..j0+RN-1 of one C^p.
//   a: stored A^p in shared memory, packed (ld = rows of stored A)
//   b: stored B^p in shared memory, packed
//   cin: packed input C^p (beta != 0), cout/ldo: output location.
// MS/NS/KS are the compile-time sizes (0 = use m/n/k).
// --------------------------------------------------------------------------
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, int RM, int RN>
__device__ __forceinline__ void micro_tile(const T *__restrict__ a, const T *__restrict__ b,
                                           const T *__restrict__ cin, T *__restrict__ cout,
                                           int ldo, int i0, int j0, int m_, int n_, int k_,
                                           T alpha, T beta)
{
    constexpr bool CA = (OPA == OP_C), CBc = (OPB == OP_C);
    constexpr int KMAX = KS ? KS : 16;
    const int m = MS ? MS : m_;
    const int n = NS ? NS : n_;
    const int k = KS ? KS : k_;
    // op(A)_{il} = a[i + m*l] (N) or a[l + k*i] (T/C); op(B)_{lj} = b[l + k*j] (N) or b[j + n*l].
    const int sa = (OPA == OP_N) ? m : 1;
    const int sb = (OPB == OP_N) ? 1 : n;
    const T *ar[RM];
    const T *bc[RN];
#pragma unroll
    for (int r = 0; r < RM; ++r) {
        const int i = min(i0 + r, m - 1);  // clamp: rows >= m are computed but never stored
        ar[r] = (OPA == OP_N) ? a + i : a + i * k;
    }
#pragma unroll
    for (int c = 0; c < RN; ++c) {
        const int j = min(j0 + c, n - 1);
        bc[c] = (OPB == OP_N) ? b + j * k : b + j;
    }
    T acc[RM][RN];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < RN; ++c) acc[r][c] = zero<T>();

#pragma unroll
    for (int l = 0; l < KMAX; ++l) {
        if (KS == 0 && l >= k) break;
        T av[RM], bv[RN];
#pragma unroll
        for (int r = 0; r < RM; ++r) av[r] = ar[r][l * sa];
#pragma unroll
        for (int c = 0; c < RN; ++c) bv[c] = bc[c][l * sb];
#pragma unroll
        for (int r = 0; r < RM; ++r)
#pragma unroll
            for (int c = 0; c < RN; ++c) mac<CA, CBc>(acc[r][c], av[r], bv[c]);
    }

    constexpr bool FULLM = MS && (MS % RM == 0);
    constexpr bool FULLN = NS && (NS % RN == 0);
#pragma unroll
    for (int c = 0; c < RN; ++c) {
        const int j = j0 + c;
        if (!FULLN && j >= n) continue;
#pragma unroll
        for (int r = 0; r < RM; ++r) {
            const int i = i0 + r;
            if (!FULLM && i >= m) continue;
            T y;
            if constexpr (B0)
                y = ax(alpha, acc[r][c]);
            else
                y = axpby(alpha, acc[r][c], beta, cin[i + m * j]);
            cout[i + (long long)ldo * j] = y;
        }
    }
}

// Threads -> (matrix q of the tile, row block, column block) work items.
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, int RM, int RN, int NT>
__device__ __forceinline__ void compute_tile_to_smem(const T *sA, const T *sB, const T *sC,
                                                     T *out, int np, const Params<T> &p)
{
    const int m = MS ? MS : p.m, n = NS ? NS : p.n, k = KS ? KS : p.k;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int CBn = (n + RN - 1) / RN;
    const int TPM = ((m + RM - 1) / RM) * CBn;
    const int items = np * TPM;
    for (int w = threadIdx.x; w < items; w += NT) {
        const int q = w / TPM;
        const int sub = w - q * TPM;
        const int rb = sub / CBn;
        const int cb = sub - rb * CBn;
        micro_tile<T, MS, NS, KS, OPA, OPB, B0, RM, RN>(sA + q * SA, sB + q * SB,
                                                         B0 ? nullptr : sC + q * SC, out + q * SC,
                                                         m, rb * RM, cb * RN, m, n, k, p.alpha,
                                                         p.beta);
    }
}

// --------------------------------------------------------------------------
// Packed strided batches: bulk async copies through an S-stage mbarrier ring.
// Preconditions (host-checked): lda = rows(A), lda2 = rows(A)*cols(A) (same for
// B, C), base pointers 16-byte aligned, batch and P multiples of the 16-byte
// alignment unit, k >= 1, alpha != 0.
// Shared memory: S stages of [A tile | B tile | C-in tile], 2 output tiles,
// S mbarriers.
// --------------------------------------------------------------------------
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, int RM, int RN, int NT>
__global__ void __launch_bounds__(NT) bulk_kernel(const Params<T> p)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int m = MS ? MS : p.m, n = NS ? NS : p.n, k = KS ? KS : p.k;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int P = p.P, S = p.S;
    const int stage_elems = P * (SA + SB + (B0 ? 0 : SC));
    T *stage0 = reinterpret_cast<T *>(smem_raw);
    T *out0 = stage0 + (long long)S * stage_elems;
    uint64_t *bars = reinterpret_cast<uint64_t *>(out0 + 2 * P * SC);

    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;
    const uint64_t pol = policy_evict_first();

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int i) {  // local tile i -> stage i % S (thread 0 only)
        const long long t = blockIdx.x + (long long)i * G;
        const long long pair0 = t * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        T *st = stage0 + (long long)(i % S) * stage_elems;
        const uint32_t ba = np * SA * (uint32_t)sizeof(T);
        const uint32_t bb = np * SB * (uint32_t)sizeof(T);
        const uint32_t bcin = B0 ? 0u : np * SC * (uint32_t)sizeof(T);
        uint64_t *bar = &bars[i % S];
        mbar_arrive_expect_tx(bar, ba + bb + bcin);
        bulk_g2s(st, p.A + pair0 * SA, ba, bar, pol);
        bulk_g2s(st + P * SA, p.B + pair0 * SB, bb, bar, pol);
        if (!B0) bulk_g2s(st + P * (SA + SB), p.C + pair0 * SC, bcin, bar, pol);
    };

    if (tid == 0)
        for (int i = 0; i < S - 1 && i < my_tiles; ++i) issue(i);

    for (int i = 0; i < my_tiles; ++i) {
        if (tid == 0 && i + S - 1 < my_tiles) issue(i + S - 1);
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        T *st = stage0 + (long long)(i % S) * stage_elems;
        T *out = out0 + (i & 1) * P * SC;
        mbar_wait(&bars[i % S], (i / S) & 1);
        compute_tile_to_smem<T, MS, NS, KS, OPA, OPB, B0, RM, RN, NT>(st, st + P * SA,
                                                                       st + P * (SA + SB), out,
                                                                       np, p);
        fence_proxy_async_smem();      // our st.shared -> visible to the bulk store
        if (tid == 0) bulk_wait_read<0>();  // store of tile i-1 has finished reading out[(i+1)&1]
        __syncthreads();               // tile i consumed (stage free), out[i&1] complete
        if (tid == 0) {
            bulk_s2g(p.C + pair0 * SC, out, np * SC * (uint32_t)sizeof(T), pol);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait<0>();
}

// --------------------------------------------------------------------------
// General strided / pointer-array batches: element-granular cp.async gathers
// into a GS-stage ring (packed stage layout identical to the bulk kernel's), C
// written from registers at its true address.
// --------------------------------------------------------------------------
constexpr int GS = 3;

template <class T, int OPA, int OPB, bool B0, int RM, int RN, int NT, bool PTR>
__global__ void __launch_bounds__(NT) gather_kernel(const Params<T> p)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int m = p.m, n = p.n, k = p.k;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int rowsA = (OPA == OP_N) ? m : k;
    const int rowsB = (OPB == OP_N) ? k : n;
    const int P = p.P;
    const int stage_elems = P * (SA + SB + (B0 ? 0 : SC));
    T *stage0 = reinterpret_cast<T *>(smem_raw);
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;

    auto issue = [&](int i) {
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        T *st = stage0 + (long long)(i % GS) * stage_elems;
        for (int e = tid; e < np * SA; e += NT) {
            const int q = e / SA, r = e - q * SA;
            const int row = r % rowsA, col = r / rowsA;
            const T *src = PTR ? p.Ap[pair0 + q] : p.A + (pair0 + q) * p.lda2;
            cp_async<sizeof(T)>(st + e, src + row + (long long)p.lda * col);
        }
        T *sb = st + P * SA;
        for (int e = tid; e < np * SB; e += NT) {
            const int q = e / SB, r = e - q * SB;
            const int row = r % rowsB, col = r / rowsB;
            const T *src = PTR ? p.Bp[pair0 + q] : p.B + (pair0 + q) * p.ldb2;
            cp_async<sizeof(T)>(sb + e, src + row + (long long)p.ldb * col);
        }
        if (!B0) {
            T *sc = st + P * (SA + SB);
            for (int e = tid; e < np * SC; e += NT) {
                const int q = e / SC, r = e - q * SC;
                const int row = r % m, col = r / m;
                const T *src = PTR ? p.Cp[pair0 + q] : p.C + (pair0 + q) * p.ldc2;
                cp_async<sizeof(T)>(sc + e, src + row + (long long)p.ldc * col);
            }
        }
    };

    for (int i = 0; i < GS - 1; ++i) {
        if (i < my_tiles) issue(i);
        cp_async_commit();
    }
    const int CBn = (n + RN - 1) / RN;
    const int TPM = ((m + RM - 1) / RM) * CBn;
    for (int i = 0; i < my_tiles; ++i) {
        if (i + GS - 1 < my_tiles) issue(i + GS - 1);
        cp_async_commit();
        cp_async_wait<GS - 1>();
        __syncthreads();
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        const T *st = stage0 + (long long)(i % GS) * stage_elems;
        const T *sA = st, *sB = st + P * SA, *sC = st + P * (SA + SB);
        const int items = np * TPM;
        for (int w = tid; w < items; w += NT) {
            const int q = w / TPM;
            const int sub = w - q * TPM;
            const int rb = sub / CBn, cb = sub - rb * CBn;
            T *cout = PTR ? p.Cp[pair0 + q] : p.C + (pair0 + q) * p.ldc2;
            micro_tile<T, 0, 0, 0, OPA, OPB, B0, RM, RN>(sA + q * SA, sB + q * SB,
                                                         B0 ? nullptr : sC + q * SC, cout, p.ldc,
                                                         rb * RM, cb * RN, m, n, k, p.alpha,
                                                         p.beta);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
}

// --------------------------------------------------------------------------
// alpha == 0 or k == 0: C <- beta*C (A, B never read), or C <- 0 when beta == 0
// (C never read).  Reading of the empty-sum / alpha = 0 case: DESIGN.md R4.
// --------------------------------------------------------------------------
__device__ __forceinline__ float scal(float b, float y) { return b * y; }
__device__ __forceinline__ double scal(double b, double y) { return b * y; }
__device__ __forceinline__ float2 scal(float2 b, float2 y)
{
    return make_float2(b.x * y.x - b.y * y.y, b.x * y.y + b.y * y.x);
}
__device__ __forceinline__ double2 scal(double2 b, double2 y)
{
    return make_double2(b.x * y.x - b.y * y.y, b.x * y.y + b.y * y.x);
}

template <class T, bool PTR, bool B0>
__global__ void __launch_bounds__(256) scale_kernel(const Params<T> p)
{
    const long long mn = (long long)p.m * p.n;
    const long long total = mn * p.batch;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long q = e / mn;
        const int r = (int)(e - q * mn);
        const int i = r % p.m, j = r / p.m;
        T *c = PTR ? p.Cp[q] : p.C + q * p.ldc2;
        T &y = c[i + (long long)p.ldc * j];
        if constexpr (B0)
            y = zero<T>();
        else
            y = scal(p.beta, y);
    }
}

}  // namespace tx
