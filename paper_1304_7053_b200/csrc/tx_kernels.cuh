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
//    by mbarriers; C is stored from registers with coalesced vector stores.
//    Persistent CTAs loop over tiles (the paper's "each CUDA
//    thread-block is used to process multiple matrices").
//  * gather_kernel -- any strided layout (padded ld/ld2, broadcast ld2 = 0,
//    unaligned bases) and the pointer-array layout: element-
//    granular cp.async (LDGSTS) gathers into the same packed stage layout, C is
//    written straight from registers.
#pragma once

#ifndef __CUDACC_RTC__
#include "tx_common.cuh"
#else
typedef unsigned long long uintptr_t;
#endif

namespace tx {

constexpr int TXK_MAX_DIM = 64;  // largest m, n, k (TX_MAX_DIM in include/txgemm.h)

// A 128-byte TMA tensor map (the CUtensorMap blob, encoded on the host by
// cuTensorMapEncodeTiled); used by the ASW bulk instances.
struct alignas(64) TmaDesc {
    unsigned long long w[16];
};

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
    const T *alpha_dev;  // device-resident alpha / beta (DEVAB kernels), else null
    const T *beta_dev;
    TmaDesc tma_a;       // ASW instances: tensor map of stored A (see bulk_kernel)
    TmaDesc tma_b;       // BSW instances: tensor map of stored B
};

// --------------------------------------------------------------------------
// Thread mapping (chosen per instance by tools/mapsearch.cpp, see
// tx_map_table.inc): each thread owns an RM x RN micro-tile of one C^p.
//   rows  i_r = rb*RM + r (RMODE 0) | rb + RB*r (RMODE 1)
//   cols  j_c = cb*RN + c (CMODE 0) | cb + CB*c (CMODE 1), then rotated by
//         q*ROTN (mod n) so neighbouring matrices hit different banks
//   lanes rb fastest (LO 0) | cb fastest (LO 1)
//   VA/VB/VC: vector width (elements) of the shared-memory accesses of A, B
//         and C along their stored-contiguous dimension.
//   S, KB: pipeline stages and stage-size target the planner uses (autotuned).
// Every mapping accumulates each output over l = 0..k-1 in ascending order, so
// all mappings (and the gather / pointer paths) give bitwise-identical results.
// --------------------------------------------------------------------------
template <int RM_, int RN_, int RMODE_, int CMODE_, int LO_, int VA_, int VB_, int VC_, int ROTN_,
          int S_ = 0, int KB_ = 0>
struct MapT {
    static constexpr int RM = RM_, RN = RN_, RMODE = RMODE_, CMODE = CMODE_, LO = LO_;
    static constexpr int VA = VA_, VB = VB_, VC = VC_, ROTN = ROTN_;
    static constexpr int S = S_;    // pipeline stages (0 = planner's choice)
    static constexpr int KB = KB_;  // stage-size target in KB (0 = default 16)
};

// Vector shared/global accesses of V consecutive elements, moved element by
// element through registers (no memcpy through pointers into local arrays,
// which made ptxas spill to local memory).
template <class T, int V>
struct Vec {
    T v[V];
};

template <class T, int V>
__device__ __forceinline__ Vec<T, V> ldv(const T *p)
{
    Vec<T, V> r;
    if constexpr (V == 1) {
        r.v[0] = *p;
    } else if constexpr (same_t<T, float>::value && V == 4) {
        const float4 u = *reinterpret_cast<const float4 *>(p);
        r.v[0] = u.x; r.v[1] = u.y; r.v[2] = u.z; r.v[3] = u.w;
    } else if constexpr (same_t<T, float>::value && V == 2) {
        const float2 u = *reinterpret_cast<const float2 *>(p);
        r.v[0] = u.x; r.v[1] = u.y;
    } else if constexpr (same_t<T, double>::value && V == 2) {
        const double2 u = *reinterpret_cast<const double2 *>(p);
        r.v[0] = u.x; r.v[1] = u.y;
    } else if constexpr (same_t<T, float2>::value && V == 2) {
        const float4 u = *reinterpret_cast<const float4 *>(p);
        r.v[0] = make_float2(u.x, u.y); r.v[1] = make_float2(u.z, u.w);
    } else {
        static_assert(V == 1, "unsupported vector width");
    }
    return r;
}

template <class T, int V>
__device__ __forceinline__ void stv(T *p, const Vec<T, V> &r)
{
    if constexpr (V == 1) {
        *p = r.v[0];
    } else if constexpr (same_t<T, float>::value && V == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
    } else if constexpr (same_t<T, float>::value && V == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(r.v[0], r.v[1]);
    } else if constexpr (same_t<T, double>::value && V == 2) {
        *reinterpret_cast<double2 *>(p) = make_double2(r.v[0], r.v[1]);
    } else if constexpr (same_t<T, float2>::value && V == 2) {
        *reinterpret_cast<float4 *>(p) = make_float4(r.v[0].x, r.v[0].y, r.v[1].x, r.v[1].y);
    } else {
        static_assert(V == 1, "unsupported vector width");
    }
}

// One micro-tile of one C^p.
//   a, b: stored A^p, B^p in shared memory, packed (ld = stored rows)
//   cin : packed input C^p in shared memory (beta != 0)
//   cout/ldo: destination of C^p (global memory, true leading dimension)
// MS/NS/KS are compile-time sizes (0 = use m_/n_/k_; then the mapping must be
// scalar, VA = VB = VC = 1).
// LDAS: leading dimension of A-N in shared memory when it is not m (the padded
// transposed copy of the TRA path); CONJA >= 0 overrides the conjugation of A.
// ASW: stored A (op T/C, k*sizeof(T) a multiple of 128 bytes) lies in shared
// memory with the 128-byte swizzle (written so by the TMA engine, or by the
// gather kernel's copies): row i of the matrix (stored column i, k elements) is
// a 128-byte line (a_rs bytes apart for each further 128 bytes of the row), and
// its 16-byte chunk c sits at chunk c ^ ((a_row0 + i) mod 8), a_row0 = the
// matrix's first line in the region.  BSW: the same for stored B with op N
// (column j of B, k elements, is line b_row0 + j; regions b_rs bytes apart).
// Lanes reading one l of 8 consecutive rows then hit 8 different chunks: no
// bank conflicts, with no transpose pass.
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, class MP, int LDAS = 0,
          int CONJA = -1, bool ASW = false, bool BSW = false>
__device__ __forceinline__ void micro_tile(const T *__restrict__ a, const T *__restrict__ b,
                                           const T *__restrict__ cin, T *__restrict__ cout,
                                           long long ldo, int rb, int cb, int q, int m_, int n_,
                                           int k_, T alpha, T beta, int a_rs = 0, int a_row0 = 0,
                                           int b_rs = 0, int b_row0 = 0)
{
    constexpr int RM = MP::RM, RN = MP::RN;
    constexpr bool CA = CONJA >= 0 ? (CONJA != 0) : (OPA == OP_C), CBc = (OPB == OP_C);
    constexpr int VA = MP::VA, VB = MP::VB, VC = MP::VC;
    constexpr int VLa = (OPA != OP_N && VA > 1) ? VA : 1;   // A vectors run along l
    constexpr int VLb = (OPB == OP_N && VB > 1) ? VB : 1;   // B vectors run along l
    constexpr int VL = VLa > VLb ? VLa : VLb;
    constexpr int KMAX = KS ? KS : TXK_MAX_DIM;
    const int m = MS ? MS : m_;
    const int n = NS ? NS : n_;
    const int k = KS ? KS : k_;
    const int RB = (m + RM - 1) / RM, CB = (n + RN - 1) / RN;
    const int lda_s = LDAS ? LDAS : m;

    // ---- rows and columns owned by this thread
    int ir[RM];
    bool rv[RM];
#pragma unroll
    for (int r = 0; r < RM; ++r) {
        const int i = MP::RMODE == 0 ? rb * RM + r : rb + RB * r;
        rv[r] = i < m;
        ir[r] = min(i, m - 1);  // rows >= m are computed but never stored
    }
    constexpr int VAr = (OPA == OP_N) ? VA : 1;  // A vectors that run along the rows
    if constexpr (MP::RMODE == 0 && (VAr > 1 || VC > 1)) {
        // vector groups start on a multiple of the vector width (m % V == 0)
        constexpr int V = VAr > VC ? VAr : VC;
        static_assert(RM % V == 0, "row vector groups");
#pragma unroll
        for (int g = 0; g < RM; g += V) {
            const int i0 = min(rb * RM + g, m - V);
#pragma unroll
            for (int t = 0; t < V; ++t) ir[g + t] = i0 + t;
        }
    }
    int jc[RN];
    bool cv[RN];
#pragma unroll
    for (int c = 0; c < RN; ++c) {
        int j = MP::CMODE == 0 ? cb * RN + c : cb + CB * c;
        cv[c] = j < n;
        j = min(j, n - 1);
        if constexpr (OPB != OP_N && VB > 1) {
            static_assert(MP::CMODE == 0 && RN % VB == 0, "column vector groups");
            j = min(cb * RN + (c / VB) * VB, n - VB) + c % VB;
        }
        if constexpr (MP::ROTN != 0) j = (j + q * MP::ROTN) % n;
        jc[c] = j;
    }

    T acc[RM][RN];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < RN; ++c) acc[r][c] = zero<T>();

#pragma unroll
    for (int l0 = 0; l0 < KMAX; l0 += VL) {
        if (KS == 0 && l0 >= k) break;
        T av[RM][VL], bv[RN][VL];
        // op(A)_{il}: a[i + m*l] (N) or a[l + k*i] (T/C)
        if constexpr (OPA == OP_N) {
#pragma unroll
            for (int g = 0; g < RM; g += VA)
#pragma unroll
                for (int t = 0; t < VL; ++t) {
                    const Vec<T, VA> u = ldv<T, VA>(a + ir[g] + lda_s * (l0 + t));
#pragma unroll
                    for (int e = 0; e < VA; ++e) av[g + e][t] = u.v[e];
                }
        } else if constexpr (ASW) {
            static_assert(OPA != OP_N && KS > 0 && (KS * sizeof(T)) % 128 == 0, "ASW");
#pragma unroll
            for (int r = 0; r < RM; ++r) {
                const char *rowp = reinterpret_cast<const char *>(a) + 128 * ir[r];
                const int x = ((ir[r] + a_row0) & 7) << 4;  // line index within the region
#pragma unroll
                for (int t = 0; t < VL; t += VLa) {
                    constexpr int ES = (int)sizeof(T);
                    const int lb = (l0 + t) * ES;  // compile-time after unrolling
                    const char *src = rowp + (lb >> 7) * a_rs + (((lb & 127) & ~15) ^ x) + (lb & 15);
                    const Vec<T, VLa> u = ldv<T, VLa>(reinterpret_cast<const T *>(src));
#pragma unroll
                    for (int e = 0; e < VLa; ++e) av[r][t + e] = u.v[e];
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < RM; ++r)
#pragma unroll
                for (int t = 0; t < VL; t += VLa) {
                    const Vec<T, VLa> u = ldv<T, VLa>(a + (l0 + t) + k * ir[r]);
#pragma unroll
                    for (int e = 0; e < VLa; ++e) av[r][t + e] = u.v[e];
                }
        }
        // op(B)_{lj}: b[l + k*j] (N) or b[j + n*l] (T/C)
        if constexpr (BSW) {
            static_assert(OPB == OP_N && KS > 0 && (KS * sizeof(T)) % 128 == 0, "BSW");
#pragma unroll
            for (int c = 0; c < RN; ++c) {
                const char *rowp = reinterpret_cast<const char *>(b) + 128 * jc[c];
                const int x = ((jc[c] + b_row0) & 7) << 4;
#pragma unroll
                for (int t = 0; t < VL; t += VLb) {
                    constexpr int ES = (int)sizeof(T);
                    const int lb = (l0 + t) * ES;
                    const char *src = rowp + (lb >> 7) * b_rs + (((lb & 127) & ~15) ^ x) + (lb & 15);
                    const Vec<T, VLb> u = ldv<T, VLb>(reinterpret_cast<const T *>(src));
#pragma unroll
                    for (int e = 0; e < VLb; ++e) bv[c][t + e] = u.v[e];
                }
            }
        } else if constexpr (OPB == OP_N) {
#pragma unroll
            for (int c = 0; c < RN; ++c)
#pragma unroll
                for (int t = 0; t < VL; t += VLb) {
                    const Vec<T, VLb> u = ldv<T, VLb>(b + (l0 + t) + k * jc[c]);
#pragma unroll
                    for (int e = 0; e < VLb; ++e) bv[c][t + e] = u.v[e];
                }
        } else {
#pragma unroll
            for (int g = 0; g < RN; g += VB)
#pragma unroll
                for (int t = 0; t < VL; ++t) {
                    const Vec<T, VB> u = ldv<T, VB>(b + jc[g] + n * (l0 + t));
#pragma unroll
                    for (int e = 0; e < VB; ++e) bv[g + e][t] = u.v[e];
                }
        }
#pragma unroll
        for (int t = 0; t < VL; ++t)
#pragma unroll
            for (int r = 0; r < RM; ++r)
#pragma unroll
                for (int c = 0; c < RN; ++c) mac<CA, CBc>(acc[r][c], av[r][t], bv[c][t]);
    }

    // ---- epilogue (the paper's axpby functors)
#pragma unroll
    for (int c = 0; c < RN; ++c) {
        if (!cv[c]) continue;
        const int j = jc[c];
#pragma unroll
        for (int g = 0; g < RM; g += VC) {
            if (!rv[g]) continue;
            const int i = ir[g];
            Vec<T, VC> y;
            if constexpr (B0) {
#pragma unroll
                for (int e = 0; e < VC; ++e) y.v[e] = ax(alpha, acc[g + e][c]);
            } else {
                const Vec<T, VC> x = ldv<T, VC>(cin + i + m * j);
#pragma unroll
                for (int e = 0; e < VC; ++e) y.v[e] = axpby(alpha, acc[g + e][c], beta, x.v[e]);
            }
            stv<T, VC>(cout + i + ldo * j, y);
        }
    }
}

// --------------------------------------------------------------------------
// FP64 tensor-core (DMMA) inner products: one WARP computes a macro-tile of C^p
// (RT x CT tiles of 8 x 8; the whole C^p when m, n <= 16) with mma.sync m8n8k4 f64.
//
// Measured on the B200 (tools/dmma_probe.py): D = A*B + C of m8n8k4 f64 is
// exactly the chain of fused multiply-adds over k = 0, 1, 2, 3 in that order,
// for every element (16384 / 16384, including inputs spread over 2^+-30), and
// runs at the DFMA rate (37 TFlop/s).  So a k-step that covers 4 consecutive
// terms of the ascending-l FMA chain of micro_tile reproduces that chain bit for
// bit, with 1 instruction per 256 FMAs instead of 8 and the operands read from
// shared memory once per warp instead of once per register micro-tile.
//
// Real (double): k-step s covers l = 4s .. 4s+3.
// Complex (double2) in real form, interleaving (re, im) along k: k' = 2l + e,
//   Cr = sum_k' A'[i][k'] B'[k'][j],  A'[2l+e] = (ar, sab*ai)[e], B'[2l+e] = (br, bi)[e]
//   Ci = sum_k' A''[i][k'] B''[k'][j], A''[2l+e] = (ar, sa*ai)[e], B''[2l+e] = (sb*bi, br)[e]
// -- exactly mac<CA,CB>'s two chains (acc.x: ar*br then sab*ai*bi; acc.y:
// ar*(sb*bi) then (sa*ai)*br), sa/sb/sab the conjugation signs.  Rows, columns
// and l past the matrix read as 0: fma(0, 0, acc) == acc (acc, started at +0,
// is never -0 in round-to-nearest), so padding changes no bit.
// Fragment layouts (probed): A 8x4 row: a = A[g][t]; B 4x8 col: b = B[t][g];
// C 8x8: {c0, c1} = C[g][2t], C[g][2t+1]; g = lane / 4, t = lane % 4.
// --------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b)
{
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

template <class T> struct MmaOk { static constexpr bool value = false; };
template <> struct MmaOk<double> { static constexpr bool value = true; };
template <> struct MmaOk<double2> { static constexpr bool value = true; };

// Warp macro-tile shape of the tensor-core path: RT x CT tiles of 8 x 8 (accumulators
// per lane: 2 * RT * CT doubles, twice that for complex), and the number of
// macro-tiles (warp work items) per matrix.
template <class T, int MS, int NS>
struct MmaShape {
    static constexpr bool CPLX = same_t<T, double2>::value;
    static constexpr int RT = (MS + 7) / 8 < 2 ? (MS + 7) / 8 : 2;
    static constexpr int CT_MAX = CPLX ? 2 : 4;
    static constexpr int CT = (NS + 7) / 8 < CT_MAX ? (NS + 7) / 8 : CT_MAX;
    static constexpr int MR = (MS + 8 * RT - 1) / (8 * RT);  // macro-tiles down the rows
    static constexpr int MC = (NS + 8 * CT - 1) / (8 * CT);  // ... and across the columns
    static constexpr int ITEMS = MR * MC;                    // warp items per matrix
};

// One macro-tile (item `it` of MmaShape::ITEMS) of C^p by the lanes of one warp.
// a, b, cin: packed stored matrices in shared memory; cout/ldo: destination.
// MS, NS, KS compile-time: <= 64 for double, <= 32 for double2.
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0>
__device__ __forceinline__ void mma_item(const T *__restrict__ a, const T *__restrict__ b,
                                         const T *__restrict__ cin, T *__restrict__ cout,
                                         long long ldo, int it, int lane, T alpha, T beta)
{
    static_assert(MmaOk<T>::value && MS > 0 && NS > 0 && KS > 0 &&
                      MS <= (same_t<T, double2>::value ? 32 : 64) &&
                      NS <= (same_t<T, double2>::value ? 32 : 64) &&
                      KS <= (same_t<T, double2>::value ? 32 : 64),
                  "mma_item: double (sizes <= 64) / double2 (sizes <= 32)");
    using SH = MmaShape<T, MS, NS>;
    constexpr bool CPLX = SH::CPLX;
    constexpr int RT = SH::RT, CT = SH::CT;
    constexpr int KSTEPS = CPLX ? (2 * KS + 3) / 4 : (KS + 3) / 4;
    const int g = lane >> 2, t = lane & 3;
    const int i0 = (it % SH::MR) * 8 * RT, j0 = (it / SH::MR) * 8 * CT;
    double acc[RT][CT][CPLX ? 2 : 1][2];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < CT; ++c)
#pragma unroll
            for (int h = 0; h < (CPLX ? 2 : 1); ++h) acc[r][c][h][0] = acc[r][c][h][1] = 0.0;

    if constexpr (CPLX) {
        constexpr bool CA = OPA == OP_C, CB = OPB == OP_C;
        const int e = t & 1;
        // lane-dependent signs of the odd (imaginary) k' entries
        const bool neg_a1 = e && !(CA != CB);  // sab = -1 unless exactly one side conjugated
        const bool neg_a2 = e && CA;           // sa
        const bool neg_b2 = !e && CB;          // sb on the bi entry (even k' of B'')
        const double2 *A2 = reinterpret_cast<const double2 *>(a);
        const double2 *B2 = reinterpret_cast<const double2 *>(b);
#pragma unroll 4
        for (int s = 0; s < KSTEPS; ++s) {
            const int l = 2 * s + (t >> 1);
            double af[RT];
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                const int i = i0 + r * 8 + g;
                double v = 0.0;
                if (i < MS && l < KS) {
                    const double *p = reinterpret_cast<const double *>(
                        OPA == OP_N ? A2 + i + MS * l : A2 + l + KS * i);
                    v = p[e];
                }
                af[r] = v;
            }
            double2 bf[CT];
#pragma unroll
            for (int c = 0; c < CT; ++c) {
                const int j = j0 + c * 8 + g;
                bf[c] = (j < NS && l < KS) ? (OPB == OP_N ? B2[l + KS * j] : B2[j + NS * l])
                                           : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                const double a1 = neg_a1 ? -af[r] : af[r];
                const double a2 = neg_a2 ? -af[r] : af[r];
#pragma unroll
                for (int c = 0; c < CT; ++c) {
                    const double b1 = e ? bf[c].y : bf[c].x;
                    const double b2 = e ? bf[c].x : (neg_b2 ? -bf[c].y : bf[c].y);
                    dmma884(acc[r][c][0][0], acc[r][c][0][1], a1, b1);
                    dmma884(acc[r][c][1][0], acc[r][c][1][1], a2, b2);
                }
            }
        }
    } else {
        const double *A1 = reinterpret_cast<const double *>(a);
        const double *B1 = reinterpret_cast<const double *>(b);
#pragma unroll 4
        for (int s = 0; s < KSTEPS; ++s) {
            const int l = 4 * s + t;
            double af[RT], bf[CT];
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                const int i = i0 + r * 8 + g;
                af[r] = (i < MS && l < KS) ? (OPA == OP_N ? A1[i + MS * l] : A1[l + KS * i]) : 0.0;
            }
#pragma unroll
            for (int c = 0; c < CT; ++c) {
                const int j = j0 + c * 8 + g;
                bf[c] = (j < NS && l < KS) ? (OPB == OP_N ? B1[l + KS * j] : B1[j + NS * l]) : 0.0;
            }
#pragma unroll
            for (int r = 0; r < RT; ++r)
#pragma unroll
                for (int c = 0; c < CT; ++c) dmma884(acc[r][c][0][0], acc[r][c][0][1], af[r], bf[c]);
        }
    }
    // epilogue: the paper's axpby functors, as in micro_tile
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const int i = i0 + r * 8 + g;
        if (i >= MS) continue;
#pragma unroll
        for (int c = 0; c < CT; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = j0 + c * 8 + 2 * t + h;
                if (j >= NS) continue;
                T x;
                if constexpr (CPLX) {
                    x = make_double2(acc[r][c][0][h], acc[r][c][1][h]);
                } else {
                    x = acc[r][c][0][h];
                }
                T y;
                if constexpr (B0) y = ax(alpha, x);
                else y = axpby(alpha, x, beta, cin[i + MS * j]);
                cout[i + ldo * j] = y;
            }
    }
}

// Threads -> (matrix q of the tile, row block, column block) work items.
template <class MP>
__device__ __forceinline__ void split_item(int sub, int RB, int CB, int &rb, int &cb)
{
    if constexpr (MP::LO == 0) {
        rb = sub % RB;
        cb = sub / RB;
    } else {
        cb = sub % CB;
        rb = sub / CB;
    }
}

// --------------------------------------------------------------------------
// Packed strided batches: bulk async copies through an S-stage mbarrier ring.
// Preconditions (host-checked): lda = rows(A), lda2 = rows(A)*cols(A) (same for
// B, C), base pointers 16-byte aligned, batch and P multiples of the 16-byte
// alignment unit, k >= 1, alpha != 0.
// Shared memory: S stages of [A tile | B tile | C-in tile] and S mbarriers.
// C^p is stored from registers straight to global memory (vectorised along the
// contiguous rows by the mapping), so no output staging is needed.
// --------------------------------------------------------------------------
// BCAST (fixed-operand batched GEMM, the paper's §9 variant):
// bit 0 = A is one matrix shared by every pair (lda2 = 0), bit 1 = same for B.
// A shared operand is loaded once per CTA into its own shared-memory region and
// is not part of the streamed stages, so a pair moves 2 matrices instead of 3.
// TRA (OPA = T/C): right after a tile lands, the threads transpose its A
// matrices into a padded N-layout copy (ld = m + 1, so both the transposing
// stores and the compute loads are bank-conflict free) and the compute reads A
// as op N (conjugation kept).  Chosen per instance by measurement: it pays off
// where the column reads of stored A hit one bank group (n = 16 with 8/16-byte
// elements).  MP must then be an N-style mapping with VA = 1.
// C <- beta*C (or 0) over pairs [pair0, pair0 + np) of a packed C, no A/B reads
// (alpha == 0 with device-resident scalars).
template <class T, int NT>
__device__ __forceinline__ void scale_packed(T *c, long long elems, T beta, bool b0)
{
    for (long long e = threadIdx.x; e < elems; e += NT) {
        if (b0) {
            c[e] = zero<T>();
        } else {
            T y = c[e];
            c[e] = axpby(zero<T>(), zero<T>(), beta, y);
        }
    }
}

// DEVAB: alpha and beta are read from device memory at run time (the paper's
// "host or device pointer"): the kernel is instantiated with
// B0 = false and decides in-kernel: alpha == 0 -> C <- beta*C without reading
// A, B (nothing when beta == 1); beta == 0 -> C is neither loaded nor read.
// ASW (OPA = T/C, k*sizeof(T) a multiple of 128 B): the A tile is loaded with a
// TMA tensor copy (p.tma_a: stored A as rows of k elements, one row per stored
// column, 128-byte swizzle) instead of a 1-D bulk copy, so the transposed reads
// of A are conflict-free without a transpose pass (see micro_tile).  Rows longer
// than 128 B are split into 128-byte regions, one box each.  BSW: the same for B
// with op N (p.tma_b, one row per stored column of B).  The swizzled regions
// start on 1024-byte boundaries (the swizzle atom); the host caps P*m (P*n) at
// 256 (the box height limit) and adds the alignment slack to the shared memory.
// MMA (double / double2, square sizes <= 16, no BCAST/TRA/DEVAB/ASW/BSW): each
// warp computes warp macro-tiles with the FP64 tensor cores (mma_item).
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, class MP, int NT,
          int BCAST = 0, bool TRA = false, bool DEVAB = false, bool ASW = false, bool BSW = false,
          bool MMA = false>
__global__ void __launch_bounds__(NT) bulk_kernel(const __grid_constant__ Params<T> p)
{
    static_assert(!MMA || (MmaOk<T>::value && BCAST == 0 && !TRA && !DEVAB && !ASW && !BSW &&
                           MS > 0 && NS > 0 && KS > 0), "MMA");
    constexpr bool BA = (BCAST & 1) != 0, BB = (BCAST & 2) != 0;
    static_assert(!TRA || (OPA != OP_N && BCAST == 0 && MS > 0 && MP::VA == 1), "TRA");
    static_assert(!DEVAB || (!B0 && !TRA && BCAST == 0), "DEVAB");
    static_assert(!ASW || (OPA != OP_N && BCAST == 0 && !TRA && !DEVAB && MS > 0 && KS > 0 &&
                           (KS * sizeof(T)) % 128 == 0), "ASW");
    static_assert(!BSW || (OPB == OP_N && BCAST == 0 && !TRA && !DEVAB && NS > 0 && KS > 0 &&
                           (KS * sizeof(T)) % 128 == 0), "BSW");
    constexpr bool SWZ = ASW || BSW;
    constexpr int ES = (int)sizeof(T);
    constexpr int NREG = SWZ ? (int)(KS * sizeof(T) / 128) : 1;  // 128-byte regions per row
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int m = MS ? MS : p.m, n = NS ? NS : p.n, k = KS ? KS : p.k;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int sSA = BA ? 0 : SA, sSB = BB ? 0 : SB;  // per-pair elements in a stage
    const int RB = (m + MP::RM - 1) / MP::RM, CB = (n + MP::RN - 1) / MP::RN;
    const int TPM = RB * CB;
    const int P = p.P, S = p.S;
    // stage: [A tile | B tile | C-in tile], byte offsets.  A swizzled tile is NREG
    // regions of P*m (P*n) 128-byte lines, each region on a 1024-byte boundary: the
    // hardware swizzle keys on address bits 7-9, which then equal the line index.
    const int a_rs = ASW ? ((P * m * 128 + 1023) & ~1023) : P * m * 128;
    const int b_rs = BSW ? ((P * n * 128 + 1023) & ~1023) : P * n * 128;
    const int bytesA = ASW ? NREG * a_rs : P * sSA * ES;
    const int offB = SWZ ? ((bytesA + 1023) & ~1023) : bytesA;
    const int offC = offB + (BSW ? NREG * b_rs : P * sSB * ES);
    const int stage_raw = offC + (B0 ? 0 : P * SC * ES);
    const int stage_elems = (SWZ ? ((stage_raw + 1023) & ~1023) : stage_raw) / ES;
    T *stage0 = reinterpret_cast<T *>(
        SWZ ? (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023
            : reinterpret_cast<uintptr_t>(smem_raw));
    T *shared_ab = stage0 + (long long)S * stage_elems;  // broadcast A then B (packed)
    constexpr int LDT = MS + 1;                          // TRA: padded transposed A
    T *atr = shared_ab + (BA ? SA : 0) + (BB ? SB : 0);
    const int tr_elems = TRA ? P * LDT * k : 0;
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        reinterpret_cast<unsigned char *>(stage0) +
        (((long long)S * stage_elems + (BA ? SA : 0) + (BB ? SB : 0) + tr_elems) * sizeof(T) + 15) /
            16 * 16);

    // Decoupled ring (build with -DTX_DEC; all but TRA, whose transposed copy is a
    // CTA-wide buffer): bars[s] = "stage s full" (the copies' bytes), empty[s] = "stage s
    // consumed" (one arrive per warp).  Thread 0 refills a stage once every warp has
    // released it, so no warp waits at a CTA barrier for the slowest one; the warps'
    // item assignment rotates by one warp per tile so a tile's partial last pass over
    // the thread block lands on each warp in turn.  Motivated by ncu (c13 beta = 0: 1.9
    // of 5.9 cycles per issued instruction were barrier stalls at the per-tile
    // __syncthreads), but an interleaved gate A/B over all 832 square instances measured
    // no net gain (median ratio 0.999, 104 instances faster and 173 slower by > 2 %,
    // c13 beta = 0 0.94x; profiles/r02s3_dec_ab/), so the default build keeps the
    // per-tile __syncthreads ring.
#ifdef TX_DEC
    constexpr bool DEC = !TRA;
#else
    constexpr bool DEC = false;
#endif
    constexpr int NW = NT / 32;
    uint64_t *empty = bars + S;
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;
    const uint64_t pol = policy_evict_first();

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&bars[s], 1);
            if (DEC) mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    grid_dep_wait();    // PDL: the prologue above overlapped the previous grid's tail
    grid_dep_launch();
    T alpha = p.alpha, beta = p.beta;
    bool b0r = B0;
    if constexpr (DEVAB) {
        alpha = *p.alpha_dev;
        beta = *p.beta_dev;
        b0r = is_zero(beta);
        if (is_zero(alpha)) {  // C <- beta*C; A and B are never read
            if (is_one(beta)) return;
            for (int i = 0; i < my_tiles; ++i) {
                const long long pair0 = (blockIdx.x + (long long)i * G) * P;
                const int np = (int)min((long long)P, p.batch - pair0);
                scale_packed<T, NT>(p.C + pair0 * SC, (long long)np * SC, beta, b0r);
            }
            return;
        }
    }
    if constexpr (BA || BB) {  // the shared operand(s), once per CTA (any alignment)
        if (BA)
            for (int e = threadIdx.x; e < SA; e += NT) shared_ab[e] = p.A[e];
        if (BB)
            for (int e = threadIdx.x; e < SB; e += NT) shared_ab[(BA ? SA : 0) + e] = p.B[e];
        __syncthreads();
    }

    auto issue = [&](int i) {  // local tile i -> stage i % S (thread 0 only)
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        T *st = stage0 + (long long)(i % S) * stage_elems;
        // ASW / BSW: a box always lands whole (rows past the batch are zero-filled)
        const uint32_t ba = BA ? 0u : (ASW ? P : np) * SA * (uint32_t)sizeof(T);
        const uint32_t bb = BB ? 0u : (BSW ? P : np) * SB * (uint32_t)sizeof(T);
        const uint32_t bcin = b0r ? 0u : np * SC * (uint32_t)sizeof(T);
        uint64_t *bar = &bars[i % S];
        char *stb = reinterpret_cast<char *>(st);
        mbar_arrive_expect_tx(bar, ba + bb + bcin);
        if constexpr (ASW) {
            if constexpr (NREG == 1) {
                tma_g2s_2d(stb, &p.tma_a, 0, (int)(pair0 * m), bar, pol);
            } else {
#pragma unroll
                for (int h = 0; h < NREG; ++h)
                    tma_g2s_3d(stb + h * a_rs, &p.tma_a, 0, h, (int)(pair0 * m), bar, pol);
            }
        } else if (!BA) {
            bulk_g2s(st, p.A + pair0 * SA, ba, bar, pol);
        }
        if constexpr (BSW) {
            if constexpr (NREG == 1) {
                tma_g2s_2d(stb + offB, &p.tma_b, 0, (int)(pair0 * n), bar, pol);
            } else {
#pragma unroll
                for (int h = 0; h < NREG; ++h)
                    tma_g2s_3d(stb + offB + h * b_rs, &p.tma_b, 0, h, (int)(pair0 * n), bar, pol);
            }
        } else if (!BB) {
            bulk_g2s(stb + offB, p.B + pair0 * SB, bb, bar, pol);
        }
        if (!b0r) bulk_g2s(stb + offC, p.C + pair0 * SC, bcin, bar, pol);
    };

    if (tid == 0)
        for (int i = 0; i < S - 1 && i < my_tiles; ++i) issue(i);

    for (int i = 0; i < my_tiles; ++i) {
        if (tid == 0 && i + S - 1 < my_tiles) {
            // tile i + S - 1 reuses the stage of tile i - 1
            if (DEC && i >= 1) mbar_wait(&empty[(i - 1) % S], ((i - 1) / S) & 1);
            issue(i + S - 1);
        }
        // rotated thread / warp index of this tile (DEC)
        const int rw = DEC ? ((tid >> 5) + i) % NW : (tid >> 5);
        const int rt = DEC ? rw * 32 + (tid & 31) : tid;
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        const T *st = stage0 + (long long)(i % S) * stage_elems;
        const T *sA = BA ? shared_ab : st;
        const T *sB = BB ? shared_ab + (BA ? SA : 0)
                         : reinterpret_cast<const T *>(reinterpret_cast<const char *>(st) + offB);
        const T *sC = reinterpret_cast<const T *>(reinterpret_cast<const char *>(st) + offC);
        T *gC = p.C + pair0 * SC;
        mbar_wait(&bars[i % S], (i / S) & 1);
        const int items = np * TPM;
        if constexpr (TRA) {
            // stored A^q is k x m (element (l, i) at l + k*i): copy to atr[q][i + LDT*l]
            for (int e = tid; e < np * SA; e += NT) {
                const int q = e / SA, r = e - q * SA;
                const int l = r % KS, i = r / KS;
                atr[q * (LDT * KS) + i + LDT * l] = sA[e];
            }
            __syncthreads();
            for (int w = tid; w < items; w += NT) {
                const int q = w / TPM;
                int rb, cb;
                split_item<MP>(w - q * TPM, RB, CB, rb, cb);
                micro_tile<T, MS, NS, KS, OP_N, OPB, B0, MP, LDT, (OPA == OP_C) ? 1 : 0>(
                    atr + q * (LDT * KS), sB + (BB ? 0 : q * SB), B0 ? nullptr : sC + q * SC,
                    gC + q * SC, m, rb, cb, q, m, n, k, p.alpha, p.beta);
            }
        } else if constexpr (MMA) {
            const int lane = tid & 31;
            constexpr int IT = MmaShape<T, (MS > 0 ? MS : 1), (NS > 0 ? NS : 1)>::ITEMS;
            for (int w = rw; w < np * IT; w += NT / 32) {
                const int q = w / IT;
                mma_item<T, MS, NS, KS, OPA, OPB, B0>(sA + q * SA, sB + q * SB,
                                                      B0 ? nullptr : sC + q * SC, gC + q * SC, m,
                                                      w - q * IT, lane, alpha, beta);
            }
        } else if (DEVAB && b0r) {  // run-time beta == 0: C is never read
            for (int w = rt; w < items; w += NT) {
                const int q = w / TPM;
                int rb, cb;
                split_item<MP>(w - q * TPM, RB, CB, rb, cb);
                micro_tile<T, MS, NS, KS, OPA, OPB, true, MP>(sA + q * SA, sB + q * SB, nullptr,
                                                              gC + q * SC, m, rb, cb, q, m, n, k,
                                                              alpha, beta);
            }
        } else if constexpr (SWZ) {
            for (int w = rt; w < items; w += NT) {
                const int q = w / TPM;
                int rb, cb;
                split_item<MP>(w - q * TPM, RB, CB, rb, cb);
                micro_tile<T, MS, NS, KS, OPA, OPB, B0, MP, 0, -1, ASW, BSW>(
                    ASW ? reinterpret_cast<const T *>(reinterpret_cast<const char *>(sA) + q * m * 128)
                        : sA + q * SA,
                    BSW ? reinterpret_cast<const T *>(reinterpret_cast<const char *>(sB) + q * n * 128)
                        : sB + q * SB,
                    B0 ? nullptr : sC + q * SC, gC + q * SC, m, rb, cb, q, m, n, k, p.alpha, p.beta,
                    a_rs, q * m, b_rs, q * n);
            }
        } else {
            for (int w = rt; w < items; w += NT) {
                const int q = w / TPM;
                int rb, cb;
                split_item<MP>(w - q * TPM, RB, CB, rb, cb);
                micro_tile<T, MS, NS, KS, OPA, OPB, B0, MP>(sA + (BA ? 0 : q * SA),
                                                            sB + (BB ? 0 : q * SB),
                                                            B0 ? nullptr : sC + q * SC,
                                                            gC + q * SC, m, rb, cb, q, m, n, k,
                                                            alpha, beta);
            }
        }
        if constexpr (DEC) {  // this warp is done with stage i % S
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[i % S]);
        } else {
            __syncthreads();  // stage i % S (and the transposed copy) fully consumed
        }
    }
}

// --------------------------------------------------------------------------
// Pointer-array batches of packed matrices (ld = rows) whose byte sizes are
// multiples of 16: per-matrix bulk async copies into the same S-stage mbarrier
// ring, issued by the 32 lanes of warp 0 (lane q copies matrices q, q+32, ...),
// with the tile's pointers prefetched one iteration ahead so the pointer loads
// never stall the issue.  A matrix whose pointer is not 16-byte aligned is
// copied synchronously by its lane instead, before lane 0 arrives on the stage's
// mbarrier (its bytes are excluded from the expected count).
// P <= 32 * PPL pairs per tile.
// --------------------------------------------------------------------------
// DEC: the decoupled ring of bulk_kernel (empty mbarriers, rotated warp items) instead of
// the per-tile __syncthreads; chosen per call by the host (pointer-array A/B, round 2).
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, class MP, int NT,
          bool MMA = false, bool DEC = false>
__global__ void __launch_bounds__(NT) bulk_ptr_kernel(const Params<T> p)
{
    constexpr int PPL = 4;  // pointer triples per lane (P <= 128)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int m = MS ? MS : p.m, n = NS ? NS : p.n, k = KS ? KS : p.k;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int RB = (m + MP::RM - 1) / MP::RM, CB = (n + MP::RN - 1) / MP::RN;
    const int TPM = RB * CB;
    const int P = p.P, S = p.S;
    const int stage_elems = P * (SA + SB + (B0 ? 0 : SC));
    T *stage0 = reinterpret_cast<T *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage0 + (long long)S * stage_elems);
    // the tile's C pointers, one slot per stage: written by warp 0 with the copies,
    // read by every thread's epilogue (no dependent global load in the compute loop)
    // decoupled ring as in bulk_kernel: empty[s] = "stage s consumed" (one arrive per warp)
    uint64_t *empty = bars + S;
    T **cptr = reinterpret_cast<T **>(bars + 2 * S);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&bars[s], 1);
            if (DEC) mbar_init(&empty[s], NT / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    grid_dep_wait();
    grid_dep_launch();

    const T *pa[PPL], *pb[PPL];
    const T *pc[PPL];
    auto load_ptrs = [&](int i) {  // warp 0: pointers of local tile i
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
#pragma unroll
        for (int r = 0; r < PPL; ++r) {
            const long long q = pair0 + lane + 32 * r;
            const bool ok = i < my_tiles && lane + 32 * r < P && q < p.batch;
            pa[r] = ok ? p.Ap[q] : nullptr;
            pb[r] = ok ? p.Bp[q] : nullptr;
            pc[r] = ok ? (const T *)p.Cp[q] : nullptr;
        }
    };
    auto issue = [&](int i) {  // warp 0: copies of local tile i into stage i % S
        T *st = stage0 + (long long)(i % S) * stage_elems;
        uint64_t *bar = &bars[i % S];
        const uint32_t ba = SA * (uint32_t)sizeof(T), bb = SB * (uint32_t)sizeof(T),
                       bc = SC * (uint32_t)sizeof(T);
        uint32_t mine = 0;
#pragma unroll
        for (int r = 0; r < PPL; ++r) {
            if (lane + 32 * r < P) cptr[(i % S) * P + lane + 32 * r] = const_cast<T *>(pc[r]);
            if (pa[r] && (((uintptr_t)pa[r] & 15) == 0)) mine += ba;
            if (pb[r] && (((uintptr_t)pb[r] & 15) == 0)) mine += bb;
            if (!B0 && pc[r] && (((uintptr_t)pc[r] & 15) == 0)) mine += bc;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        // (1) matrices whose pointer is not 16-byte aligned: synchronous copies,
        // completed by every lane BEFORE lane 0's arrive (release) so that a thread
        // passing mbar_wait (acquire) sees them -- even when the whole tile is
        // unaligned and the expected byte count is 0.  The async-proxy fence
        // orders these generic writes before later bulk copies into the stage.
        bool sync_copied = false;
#pragma unroll
        for (int r = 0; r < PPL; ++r) {
            const int q = lane + 32 * r;
            auto copy_sync = [&](T *dst, const T *src, int elems) {
                if (!src || ((uintptr_t)src & 15) == 0) return;
                for (int e = 0; e < elems; ++e) dst[e] = src[e];
                sync_copied = true;
            };
            copy_sync(st + q * SA, pa[r], SA);
            copy_sync(st + P * SA + q * SB, pb[r], SB);
            if (!B0) copy_sync(st + P * (SA + SB) + q * SC, pc[r], SC);
        }
        if (sync_copied) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(bar, mine);
        // (2) the aligned matrices: one bulk async copy each, counted on the barrier
#pragma unroll
        for (int r = 0; r < PPL; ++r) {
            const int q = lane + 32 * r;
            auto copy_async = [&](T *dst, const T *src, uint32_t bytes) {
                if (src && ((uintptr_t)src & 15) == 0) bulk_g2s(dst, src, bytes, bar, pol);
            };
            copy_async(st + q * SA, pa[r], ba);
            copy_async(st + P * SA + q * SB, pb[r], bb);
            if (!B0) copy_async(st + P * (SA + SB) + q * SC, pc[r], bc);
        }
    };

    if (warp == 0) {
        for (int i = 0; i < S - 1 && i < my_tiles; ++i) {
            load_ptrs(i);
            issue(i);
        }
        load_ptrs(S - 1);
    }
    for (int i = 0; i < my_tiles; ++i) {
        if (warp == 0 && i + S - 1 < my_tiles) {
            // tile i + S - 1 reuses the stage (and C-pointer slots) of tile i - 1
            if (DEC && i >= 1) mbar_wait(&empty[(i - 1) % S], ((i - 1) / S) & 1);
            issue(i + S - 1);
            load_ptrs(i + S);  // consumed next iteration; latency overlaps this tile's compute
        }
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        const T *st = stage0 + (long long)(i % S) * stage_elems;
        const T *sA = st, *sB = st + P * SA, *sC = st + P * (SA + SB);
        const int rw = DEC ? (warp + i) % (NT / 32) : warp;  // rotated warp / thread index
        const int rt = rw * 32 + lane;
        mbar_wait(&bars[i % S], (i / S) & 1);
        if constexpr (MMA) {  // FP64 tensor cores: one warp per macro-tile
            constexpr int IT = MmaShape<T, (MS > 0 ? MS : 1), (NS > 0 ? NS : 1)>::ITEMS;
            for (int w = rw; w < np * IT; w += NT / 32) {
                const int q = w / IT;
                mma_item<T, MS, NS, KS, OPA, OPB, B0>(sA + q * SA, sB + q * SB,
                                                      B0 ? nullptr : sC + q * SC,
                                                      cptr[(i % S) * P + q], p.ldc, w - q * IT,
                                                      lane, p.alpha, p.beta);
            }
        } else {
            const int items = np * TPM;
            for (int w = rt; w < items; w += NT) {
                const int q = w / TPM;
                int rb, cb;
                split_item<MP>(w - q * TPM, RB, CB, rb, cb);
                micro_tile<T, MS, NS, KS, OPA, OPB, B0, MP>(sA + q * SA, sB + q * SB,
                                                            B0 ? nullptr : sC + q * SC,
                                                            cptr[(i % S) * P + q], p.ldc, rb, cb, q, m,
                                                            n, k, p.alpha, p.beta);
            }
        }
        if constexpr (DEC) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[i % S]);
        } else {
            __syncthreads();
        }
    }
}

// --------------------------------------------------------------------------
// General strided / pointer-array batches: element-granular cp.async gathers
// into a GS-stage ring (packed stage layout identical to the bulk kernel's), C
// written from registers at its true address.
// --------------------------------------------------------------------------
constexpr int GS = 3;  // gather ring depth (2 when three stages of one tile do not fit)

// V16: matrices are packed (ld = rows) with byte sizes that are multiples of 16;
// they are moved in 16-byte chunks (a chunk whose source is not 16-byte aligned
// falls back to element copies).
// PTR: the tile's matrix pointers are staged in shared memory (GS slots of
// 3 x P pointers, slot = tile % GS).  Each thread loads the pointers of tile
// i+GS+1 into registers at the end of iteration i and stores them one full
// iteration later, so the dependent pointer loads never stall a copy issue.
// The host caps P at 128 (3 x P <= 4 x NT pointer registers).
// ASWG: op(A) = T/C with k*sizeof(T) a multiple of 128 B: the copies of A are
// placed in the 128-byte-swizzled layout of micro_tile's ASW accessor (the
// destination address of each chunk / element is simply computed that way), so
// the transposed reads of A are conflict-free at no extra cost.  BSWG: the same
// for B with op N (its columns are the k-contiguous lines).
template <class T, int MS, int NS, int KS, int OPA, int OPB, bool B0, class MP, int NT, bool PTR,
          bool V16 = false, bool DEVAB = false, bool ASWG = false, bool BSWG = false,
          bool MMA = false>
__global__ void __launch_bounds__(NT) gather_kernel(const Params<T> p)
{
    static_assert(!MMA || (MmaOk<T>::value && !DEVAB && !ASWG && !BSWG && MS > 0 && NS > 0 &&
                           KS > 0), "MMA");
    static_assert(!DEVAB || !B0, "DEVAB");
    static_assert(!ASWG || (OPA != OP_N && KS > 0 && (KS * sizeof(T)) % 128 == 0 && !DEVAB), "ASWG");
    static_assert(!BSWG || (OPB == OP_N && KS > 0 && (KS * sizeof(T)) % 128 == 0 && !DEVAB), "BSWG");
    constexpr int PR = 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int m = MS ? MS : p.m, n = NS ? NS : p.n, k = KS ? KS : p.k;
    const int SA = m * k, SB = k * n, SC = m * n;
    const int rowsA = (OPA == OP_N) ? m : k;
    const int rowsB = (OPB == OP_N) ? k : n;
    const int P = p.P;
    const int gs = p.S;  // ring depth (3, or 2 when three stages of the tile do not fit)
    // operand regions of a stage start on 16-byte boundaries, so P needs no alignment
    // unit (a matrix whose elements are vector-read has a size that is a multiple of
    // the vector width; host: plan_tiles with bulk = false)
    constexpr int E16 = 16 / (int)sizeof(T) > 0 ? 16 / (int)sizeof(T) : 1;  // elements per 16 B
    const int oB = (P * SA + E16 - 1) / E16 * E16;
    const int oC = oB + (P * SB + E16 - 1) / E16 * E16;
    const int stage_elems = oC + (B0 ? 0 : (P * SC + E16 - 1) / E16 * E16);
    T *stage0 = reinterpret_cast<T *>(smem_raw);
    const T **ptab = reinterpret_cast<const T **>(
        smem_raw + (((long long)gs * stage_elems * sizeof(T) + 15) & ~15ll));
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int my_tiles = (p.ntiles - (int)blockIdx.x + G - 1) / G;
    const int a_rs = P * m * 128;  // ASWG: bytes between the 128-byte regions of the A tile
    // ASWG: byte offset in the A tile of byte pb of stored A^q (packed k x m)
    const int b_rs = P * n * 128;  // BSWG: the same for the B tile
    // ASWG / BSWG: byte offset in the A (B) tile of byte pb of stored A^q (B^q),
    // packed k x m (k x n); lines = stored columns
    auto swz = [&](int q, int pb, int cols, int rs) -> int {
        const int rb = k * (int)sizeof(T);
        const int i = pb / rb, lb = pb - i * rb, line = q * cols + i;
        return (lb >> 7) * rs + line * 128 + ((((lb & 127) >> 4) ^ (line & 7)) << 4) + (lb & 15);
    };

    // ---- pointer staging (PTR)
    const T *preg[PR];
    auto load_regs = [&](int j) {
        const long long pair0 = (blockIdx.x + (long long)j * G) * P;
#pragma unroll
        for (int t = 0; t < PR; ++t) {
            const int idx = tid + t * NT;
            const int which = idx / P, q = idx - which * P;
            const bool ok = PTR && j < my_tiles && which < 3 && pair0 + q < p.batch;
            const T *const *arr = which == 0 ? p.Ap : (which == 1 ? p.Bp : (const T *const *)p.Cp);
            preg[t] = ok ? arr[pair0 + q] : nullptr;
        }
    };
    auto store_regs = [&](int j) {
        const int slot = j % gs;
#pragma unroll
        for (int t = 0; t < PR; ++t) {
            const int idx = tid + t * NT;
            if (idx < 3 * P) ptab[slot * 3 * P + idx] = preg[t];
        }
    };
    auto ptr_of = [&](int tile, int which, int q, const T *base, long long ld2,
                      long long pair0) -> const T * {
        if constexpr (PTR) return ptab[(tile % gs) * 3 * P + which * P + q];
        else return base + (pair0 + q) * ld2;
    };

    auto chunks16 = [&](int tile, int which, T *dst0, int elems, int np, long long pair0,
                        const T *base, long long ld2) {
        const int ch = elems * (int)sizeof(T) / 16;  // chunks per matrix
        for (int e = tid; e < np * ch; e += NT) {
            const int q = e / ch, c = e - q * ch;
            const char *src =
                reinterpret_cast<const char *>(ptr_of(tile, which, q, base, ld2, pair0)) + 16 * c;
            char *dst = (ASWG && which == 0)   ? reinterpret_cast<char *>(dst0) + swz(q, 16 * c, m, a_rs)
                        : (BSWG && which == 1) ? reinterpret_cast<char *>(dst0) + swz(q, 16 * c, n, b_rs)
                                               : reinterpret_cast<char *>(dst0 + (long long)q * elems) + 16 * c;
            if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                cp_async16_cg(dst, src);
            } else {
#pragma unroll
                for (int b = 0; b < 16; b += (int)sizeof(T)) cp_async<sizeof(T)>(dst + b, src + b);
            }
        }
    };
    auto elems = [&](int tile, int which, T *dst0, int se, int rows, int ld, int np,
                     long long pair0, const T *base, long long ld2) {
        for (int e = tid; e < np * se; e += NT) {
            const int q = e / se, r = e - q * se;
            const int row = r % rows, col = r / rows;
            const T *src = ptr_of(tile, which, q, base, ld2, pair0);
            T *dst = (ASWG && which == 0)
                         ? reinterpret_cast<T *>(reinterpret_cast<char *>(dst0) +
                                                 swz(q, r * (int)sizeof(T), m, a_rs))
                     : (BSWG && which == 1)
                         ? reinterpret_cast<T *>(reinterpret_cast<char *>(dst0) +
                                                 swz(q, r * (int)sizeof(T), n, b_rs))
                         : dst0 + e;
            cp_async<sizeof(T)>(dst, src + row + (long long)ld * col);
        }
    };
    bool b0r = B0;
    auto issue = [&](int i) {
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        T *st = stage0 + (long long)(i % gs) * stage_elems;
        if constexpr (V16) {
            chunks16(i, 0, st, SA, np, pair0, p.A, p.lda2);
            chunks16(i, 1, st + oB, SB, np, pair0, p.B, p.ldb2);
            if (!b0r) chunks16(i, 2, st + oC, SC, np, pair0, p.C, p.ldc2);
        } else {
            elems(i, 0, st, SA, rowsA, p.lda, np, pair0, p.A, p.lda2);
            elems(i, 1, st + oB, SB, rowsB, p.ldb, np, pair0, p.B, p.ldb2);
            if (!b0r) elems(i, 2, st + oC, SC, m, p.ldc, np, pair0, p.C, p.ldc2);
        }
    };

    grid_dep_wait();
    grid_dep_launch();
    T alpha = p.alpha, beta = p.beta;
    if constexpr (DEVAB) {  // device-resident alpha / beta: decided here (see bulk_kernel)
        alpha = *p.alpha_dev;
        beta = *p.beta_dev;
        b0r = is_zero(beta);
        if (is_zero(alpha)) {
            if (is_one(beta)) return;
            for (int i = 0; i < my_tiles; ++i) {
                const long long pair0 = (blockIdx.x + (long long)i * G) * P;
                const int np = (int)min((long long)P, p.batch - pair0);
                for (int e = tid; e < np * SC; e += NT) {
                    const int q = e / SC, r = e - q * SC;
                    T *c = (PTR ? p.Cp[pair0 + q] : p.C + (pair0 + q) * p.ldc2) + r % m +
                           (long long)p.ldc * (r / m);
                    *c = b0r ? zero<T>() : axpby(zero<T>(), zero<T>(), beta, *c);
                }
            }
            return;
        }
    }
    if constexpr (PTR) {
        for (int j = 0; j < gs; ++j) {
            load_regs(j);
            store_regs(j);
        }
        load_regs(gs);
        __syncthreads();
    }
    for (int i = 0; i < gs - 1; ++i) {
        if (i < my_tiles) issue(i);
        cp_async_commit();
    }
    const int RB = (m + MP::RM - 1) / MP::RM, CB = (n + MP::RN - 1) / MP::RN;
    const int TPM = RB * CB;
    for (int i = 0; i < my_tiles; ++i) {
        if (i + gs - 1 < my_tiles) issue(i + gs - 1);
        cp_async_commit();
        if (gs == 3) cp_async_wait<2>(); else cp_async_wait<1>();
        __syncthreads();
        const long long pair0 = (blockIdx.x + (long long)i * G) * P;
        const int np = (int)min((long long)P, p.batch - pair0);
        const T *st = stage0 + (long long)(i % gs) * stage_elems;
        const T *sA = st, *sB = st + oB, *sC = st + oC;
        const int items = MMA ? 0 : np * TPM;
        if constexpr (MMA) {  // FP64 tensor cores: one warp per macro-tile
            const int warp = tid >> 5, lane = tid & 31;
            constexpr int IT = MmaShape<T, (MS > 0 ? MS : 1), (NS > 0 ? NS : 1)>::ITEMS;
            for (int w = warp; w < np * IT; w += NT / 32) {
                const int q = w / IT;
                T *cout = PTR ? const_cast<T *>(ptab[(i % gs) * 3 * P + 2 * P + q])
                              : p.C + (pair0 + q) * p.ldc2;
                mma_item<T, MS, NS, KS, OPA, OPB, B0>(sA + q * SA, sB + q * SB,
                                                      B0 ? nullptr : sC + q * SC, cout, p.ldc,
                                                      w - q * IT, lane, alpha, beta);
            }
        }
        for (int w = tid; w < items; w += NT) {
            const int q = w / TPM;
            int rb, cb;
            split_item<MP>(w - q * TPM, RB, CB, rb, cb);
            T *cout = PTR ? const_cast<T *>(ptab[(i % gs) * 3 * P + 2 * P + q])
                          : p.C + (pair0 + q) * p.ldc2;
            if (DEVAB && b0r)
                micro_tile<T, MS, NS, KS, OPA, OPB, true, MP>(sA + q * SA, sB + q * SB, nullptr,
                                                              cout, p.ldc, rb, cb, q, m, n, k,
                                                              alpha, beta);
            else if constexpr (ASWG || BSWG)
                micro_tile<T, MS, NS, KS, OPA, OPB, B0, MP, 0, -1, ASWG, BSWG>(
                    ASWG ? reinterpret_cast<const T *>(reinterpret_cast<const char *>(sA) + q * m * 128)
                         : sA + q * SA,
                    BSWG ? reinterpret_cast<const T *>(reinterpret_cast<const char *>(sB) + q * n * 128)
                         : sB + q * SB,
                    B0 ? nullptr : sC + q * SC, cout, p.ldc, rb, cb, q, m, n, k, alpha, beta, a_rs,
                    q * m, b_rs, q * n);
            else
                micro_tile<T, MS, NS, KS, OPA, OPB, B0, MP>(sA + q * SA, sB + q * SB,
                                                         B0 ? nullptr : sC + q * SC, cout, p.ldc,
                                                         rb, cb, q, m, n, k, alpha, beta);
        }
        __syncthreads();
        if constexpr (PTR) {  // slot i % gs is free: pointers of tile i + gs
            store_regs(i + gs);
            load_regs(i + gs + 1);
            __syncthreads();
        }
    }
    cp_async_wait<0>();
}

// --------------------------------------------------------------------------
// Tiny square matrices (n <= 2), packed and 16-byte aligned: register-direct.
// A pair's matrices are 4..64 bytes, so staging them through shared memory buys
// nothing (no reuse across threads) and the kernel is all latency: every thread
// owns G consecutive pairs (G*n*n*sizeof(T) a multiple of 16 bytes), loads its
// A, B (C) bytes with 16-byte streaming loads straight into registers -- all of
// a unit's loads in flight at once, the next unit's issued before this one is
// computed -- computes the n x n products with the same ascending-l FMA chain
// and epilogue as micro_tile (so results are bitwise identical to the other
// kernels), and stores C with 16-byte streaming stores.  The last batch % G
// pairs are done element by element by the first threads.
// --------------------------------------------------------------------------
template <class T, int N>
struct DirectShape {
    static constexpr int E = N * N;                                      // elements per matrix
    static constexpr int ES = (int)sizeof(T);
    static constexpr int G = E * ES >= 16 ? 1 : 16 / (E * ES);           // pairs per unit
    static constexpr int CH = G * E * ES / 16;                           // 16-byte chunks per operand
    static_assert((G * E * ES) % 16 == 0, "direct unit must be whole 16-byte chunks");
};

__device__ __forceinline__ uint4 ld_stream16(const void *p)
{
    uint4 r;
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream16(void *p, uint4 v)
{
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// One pair: c[i + N*j] <- alpha * sum_l op(a)_il op(b)_lj (+ beta * c[i + N*j]).
template <class T, int N, int OPA, int OPB, bool B0>
__device__ __forceinline__ void direct_pair(const T *a, const T *b, T *c, T alpha, T beta)
{
    constexpr bool CA = OPA == OP_C, CB = OPB == OP_C;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
            T acc = zero<T>();
#pragma unroll
            for (int l = 0; l < N; ++l)
                mac<CA, CB>(acc, OPA == OP_N ? a[i + N * l] : a[l + N * i],
                            OPB == OP_N ? b[l + N * j] : b[j + N * l]);
            c[i + N * j] = B0 ? ax(alpha, acc) : axpby(alpha, acc, beta, c[i + N * j]);
        }
}

template <class T, int N, int OPA, int OPB, bool B0, int NT>
__global__ void __launch_bounds__(NT) direct_kernel(const __grid_constant__ Params<T> p)
{
    using SH = DirectShape<T, N>;
    constexpr int E = SH::E, G = SH::G, CH = SH::CH;
    grid_dep_wait();
    grid_dep_launch();
    const T alpha = p.alpha, beta = p.beta;
    const long long units = p.batch / G;
    const long long stride = (long long)gridDim.x * NT;
    const uint4 *gA = reinterpret_cast<const uint4 *>(p.A);
    const uint4 *gB = reinterpret_cast<const uint4 *>(p.B);
    uint4 *gC = reinterpret_cast<uint4 *>(p.C);
    for (long long u = (long long)blockIdx.x * NT + threadIdx.x; u < units; u += 2 * stride) {
        // two units per trip, all loads issued before any arithmetic
        const long long u2 = u + stride;
        const bool two = u2 < units;
        T a[2][G * E], b[2][G * E], c[2][G * E];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long uu = h ? (two ? u2 : u) : u;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                reinterpret_cast<uint4 *>(a[h])[q] = ld_stream16(gA + uu * CH + q);
                reinterpret_cast<uint4 *>(b[h])[q] = ld_stream16(gB + uu * CH + q);
                if constexpr (!B0) reinterpret_cast<uint4 *>(c[h])[q] = ld_stream16(gC + uu * CH + q);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h == 1 && !two) break;
#pragma unroll
            for (int g = 0; g < G; ++g)
                direct_pair<T, N, OPA, OPB, B0>(a[h] + g * E, b[h] + g * E, c[h] + g * E, alpha,
                                                 beta);
            const long long uu = h ? u2 : u;
#pragma unroll
            for (int q = 0; q < CH; ++q) st_stream16(gC + uu * CH + q, reinterpret_cast<uint4 *>(c[h])[q]);
        }
    }
    // the last batch % G pairs, one per thread of the first block
    const long long tail0 = units * G;
    if (blockIdx.x == 0 && tail0 + threadIdx.x < p.batch) {
        const long long q = tail0 + threadIdx.x;
        T a[E], b[E], c[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            a[e] = p.A[q * E + e];
            b[e] = p.B[q * E + e];
            if constexpr (!B0) c[e] = p.C[q * E + e];
        }
        direct_pair<T, N, OPA, OPB, B0>(a, b, c, alpha, beta);
#pragma unroll
        for (int e = 0; e < E; ++e) p.C[q * E + e] = c[e];
    }
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

template <class T, bool PTR, bool B0, bool DEVAB = false>
__global__ void __launch_bounds__(256) scale_kernel(const Params<T> p)
{
    grid_dep_wait();
    grid_dep_launch();
    T beta = p.beta;
    bool b0r = B0;
    if constexpr (DEVAB) {  // k == 0 with device-resident beta
        beta = *p.beta_dev;
        if (is_one(beta)) return;
        b0r = is_zero(beta);
    }
    const long long mn = (long long)p.m * p.n;
    const long long total = mn * p.batch;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long q = e / mn;
        const int r = (int)(e - q * mn);
        const int i = r % p.m, j = r / p.m;
        T *c = PTR ? p.Cp[q] : p.C + q * p.ldc2;
        T &y = c[i + (long long)p.ldc * j];
        if (b0r)
            y = zero<T>();
        else
            y = scal(beta, y);
    }
}

}  // namespace tx
