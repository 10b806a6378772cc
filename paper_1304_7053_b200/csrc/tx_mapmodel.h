// tx_mapmodel.h -- shared-memory / issue model of the batched-GEMM thread mapping.
// Host C++ used by two clients: tools/mapsearch.cpp (offline exhaustive search that
// generated csrc/tx_map_table.inc) and tx_jit.cu (a compact search for the
// runtime-specialised instances: non-square shapes, pointer arrays, sizes 17-32).
//
// A mapping assigns thread (matrix q of the tile, row block rb, column block cb)
// an RM x RN micro-tile; RMODE/CMODE choose blocked or interleaved rows/cols,
// ROTN rotates a thread's columns by q*ROTN (mod N), LO picks which of rb/cb is
// the fastest-varying lane index, VA/VB/VC are the vector widths (elements) of
// the A/B/C shared-memory accesses.  Cost: per warp instruction, lanes form
// phases of 128/bytes lanes; a phase costs the max over the 32 banks of the
// distinct 4-byte words it requests; plus the 128-byte lines touched by the
// global C stores.
#pragma once

#include <algorithm>
#include <vector>

namespace txmodel {

struct Map {
    int RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN;
};

inline int blocks(int n, int r) { return (n + r - 1) / r; }

inline int wavefronts(const long *addr, int nwords, const bool *act)
{
    const int lpp = 32 / nwords;
    int total = 0;
    for (int p0 = 0; p0 < 32; p0 += lpp) {
        long words[32][32];
        int cnt[32] = {0};
        bool any = false;
        for (int ln = p0; ln < p0 + lpp; ++ln) {
            if (!act[ln]) continue;
            any = true;
            for (int w = 0; w < nwords; ++w) {
                long wd = addr[ln] + w;
                int b = (int)(((wd % 32) + 32) % 32);
                bool seen = false;
                for (int t = 0; t < cnt[b]; ++t)
                    if (words[b][t] == wd) { seen = true; break; }
                if (!seen) words[b][cnt[b]++] = wd;
            }
        }
        if (!any) continue;
        int mx = 0;
        for (int b = 0; b < 32; ++b) mx = std::max(mx, cnt[b]);
        total += mx;
    }
    return total;
}

struct Inst {
    int es, M, N, K;
    char opa, opb;  // 'N' or 'T' (C behaves like T for addressing)
    bool b0;
    // A read as op N from a padded copy (the TRA path of bulk_kernel): leading
    // dimension ldas and per-matrix stride sas in elements (0 = packed M, M*K)
    int ldas = 0, sas = 0;
    // A (op T) in the TMA 128-byte-swizzled layout of the ASW path: row i of matrix
    // q is 128-byte line q*M + i of each 128-byte region, chunk c at c ^ (line % 8)
    bool asw = false;
    bool bsw = false;  // B (op N) likewise: column j of matrix q is line q*N + j
};

inline bool valid(const Inst &s, const Map &m)
{
    const int SA = s.M * s.K, SB = s.K * s.N, SC = s.M * s.N;
    for (int v : {m.VA, m.VB, m.VC})
        if (v * s.es > 16) return false;
    const int RB = blocks(s.M, m.RM), CB = blocks(s.N, m.RN);
    if (m.RM * RB - s.M >= m.RM || m.RN * CB - s.N >= m.RN) return false;
    if (m.VA > 1) {
        if (SA % m.VA || s.ldas) return false;  // the padded copy has an odd ld
        if (s.opa == 'N') {
            if (m.RMODE != 0 || m.RM % m.VA || s.M % m.VA) return false;
        } else if (s.K % m.VA)
            return false;
    }
    if (m.VB > 1) {
        if (SB % m.VB) return false;
        if (s.opb == 'N') {
            if (s.K % m.VB) return false;
        } else if (m.CMODE != 0 || m.RN % m.VB || s.N % m.VB || m.ROTN % m.VB)
            return false;
    }
    if (m.VC > 1) {
        if (m.RMODE != 0 || m.RM % m.VC || s.M % m.VC || SC % m.VC) return false;
    }
    if (m.ROTN >= s.N && m.ROTN) return false;
    return true;
}

struct Cost {
    double wf, ninst;
    int regs;
};

inline Cost cost(const Inst &s, const Map &m, int P)
{
    const int M = s.M, N = s.N, K = s.K, wpe = s.es / 4;
    const int SA = M * K, SB = K * N, SC = M * N;
    const int RB = blocks(M, m.RM), CB = blocks(N, m.RN), tpm = RB * CB;
    const int items = P * tpm;
    const int nwarps = (items + 31) / 32;
    const int VLa = (s.opa != 'N' && m.VA > 1) ? m.VA : 1;
    const int VLb = (s.opb == 'N' && m.VB > 1) ? m.VB : 1;
    const int VL = std::max(VLa, VLb);
    Cost c{0, 0, 0};
    if (K % VL) {
        c.wf = 1e9;
        return c;
    }
    const long A0 = 0, B0 = (long)P * SA, C0 = (long)P * (SA + SB);
    long addr[32];
    bool act[32];
    int q[32], rb[32], cb[32];
    long wf = 0, ni = 0;
    for (int wi = 0; wi < nwarps; ++wi) {
        for (int ln = 0; ln < 32; ++ln) {
            int w = wi * 32 + ln;
            act[ln] = w < items;
            q[ln] = w / tpm;
            int sub = w % tpm;
            if (m.LO == 0) {
                rb[ln] = sub % RB;
                cb[ln] = sub / RB;
            } else {
                cb[ln] = sub % CB;
                rb[ln] = sub / CB;
            }
        }
        auto row = [&](int ln, int r) {
            int i = m.RMODE == 0 ? rb[ln] * m.RM + r : rb[ln] + RB * r;
            return std::min(i, M - 1);
        };
        auto col = [&](int ln, int cc) {
            int j = m.CMODE == 0 ? cb[ln] * m.RN + cc : cb[ln] + CB * cc;
            j = std::min(j, N - 1);
            if (m.ROTN) j = (j + q[ln] * m.ROTN) % N;
            return j;
        };
        for (int l0 = 0; l0 < K; l0 += VL) {
            // A
            if (s.opa == 'N') {
                const int v = m.VA;
                for (int g = 0; g < m.RM; g += v)
                    for (int l = l0; l < l0 + VL; ++l) {
                        const long sa = s.sas ? s.sas : SA, lda_s = s.ldas ? s.ldas : M;
                        for (int ln = 0; ln < 32; ++ln)
                            addr[ln] = (A0 + (long)q[ln] * sa + row(ln, g) + lda_s * l) * wpe;
                        wf += wavefronts(addr, v * wpe, act);
                        ++ni;
                    }
            } else {
                const int v = VLa;
                for (int r = 0; r < m.RM; ++r)
                    for (int l = l0; l < l0 + VL; l += v) {
                        for (int ln = 0; ln < 32; ++ln) {
                            if (s.asw) {
                                const long line = (long)q[ln] * M + row(ln, r);
                                const long lb = (long)l * s.es, c = lb % 128;
                                const long byte = (lb / 128) * (long)P * M * 128 + line * 128 +
                                                  (((c / 16) ^ (line % 8)) * 16) + c % 16;
                                addr[ln] = A0 + byte / 4;
                            } else {
                                addr[ln] = (A0 + (long)q[ln] * SA + l + (long)K * row(ln, r)) * wpe;
                            }
                        }
                        wf += wavefronts(addr, v * wpe, act);
                        ++ni;
                    }
            }
            // B
            if (s.opb == 'N') {
                const int v = VLb;
                for (int cc = 0; cc < m.RN; ++cc)
                    for (int l = l0; l < l0 + VL; l += v) {
                        for (int ln = 0; ln < 32; ++ln) {
                            if (s.bsw) {
                                const long line = (long)q[ln] * N + col(ln, cc);
                                const long lb = (long)l * s.es, c = lb % 128;
                                const long byte = (lb / 128) * (long)P * N * 128 + line * 128 +
                                                  (((c / 16) ^ (line % 8)) * 16) + c % 16;
                                addr[ln] = B0 * wpe + byte / 4;
                            } else {
                                addr[ln] = (B0 + (long)q[ln] * SB + l + (long)K * col(ln, cc)) * wpe;
                            }
                        }
                        wf += wavefronts(addr, v * wpe, act);
                        ++ni;
                    }
            } else {
                const int v = m.VB;
                for (int g = 0; g < m.RN; g += v)
                    for (int l = l0; l < l0 + VL; ++l) {
                        for (int ln = 0; ln < 32; ++ln)
                            addr[ln] = (B0 + (long)q[ln] * SB + col(ln, g) + (long)N * l) * wpe;
                        wf += wavefronts(addr, v * wpe, act);
                        ++ni;
                    }
            }
        }
        // epilogue: the beta != 0 C-in reads touch shared memory; C is stored straight
        // to global memory, costed as the number of distinct 128-byte lines each store
        // instruction touches (L1TEX wavefronts; fewer lines = better coalescing).
        for (int cc = 0; cc < m.RN; ++cc)
            for (int r = 0; r < m.RM; r += m.VC) {
                if (!s.b0) {
                    for (int ln = 0; ln < 32; ++ln)
                        addr[ln] = (C0 + (long)q[ln] * SC + row(ln, r) + (long)M * col(ln, cc)) * wpe;
                    wf += wavefronts(addr, m.VC * wpe, act);
                    ++ni;
                }
                long lines[32];
                int nl = 0;
                for (int ln = 0; ln < 32; ++ln) {
                    if (!act[ln]) continue;
                    long b0 = ((long)q[ln] * SC + row(ln, r) + (long)M * col(ln, cc)) * s.es;
                    for (long bb = b0 / 128; bb <= (b0 + m.VC * s.es - 1) / 128; ++bb) {
                        bool seen = false;
                        for (int t = 0; t < nl; ++t)
                            if (lines[t] == bb) { seen = true; break; }
                        if (!seen && nl < 32) lines[nl++] = bb;
                    }
                }
                wf += nl;
                ++ni;
            }
    }
    c.wf = (double)wf / P;
    c.ninst = (double)ni / P;
    c.regs = m.RM * m.RN * wpe + (m.RM + m.RN) * VL * wpe + 24;
    return c;
}


inline int pairs_for(int tpm)
{
    const int NT = 128;
    const int ppass = std::max(1, NT / tpm);
    return std::max(ppass, (8 * 32 + tpm - 1) / tpm);
}

// Predicted cycles per pair per SM: max(HBM, shared memory, FP pipe, issue), the
// issue rate calibrated on ncu (r01: ~2.2 warp-instructions/clock/SM at 8-12 warps).
struct Choice {
    Map map;
    int S;
    double pred, wf;
};

inline double predict(const Inst &s, const Map &m, const Cost &c, int S, bool cplx, int &ok)
{
    const int M = s.M, N = s.N, K = s.K;
    const int tpm = blocks(M, m.RM) * blocks(N, m.RN);
    const int in_bytes = (M * K + K * N + (s.b0 ? 0 : M * N)) * s.es;
    const double pair_bytes = (double)(M * K + K * N + M * N * (s.b0 ? 1 : 2)) * s.es;
    const int ppass = std::max(1, 128 / tpm);
    const int passes = std::max(1, 16384 / std::max(1, ppass * in_bytes));
    const long stage = (long)ppass * passes * std::max(in_bytes, 16);
    const int ctas = (int)std::min<long>(16, (225 * 1024L) / (S * stage + 64));
    ok = ctas >= 1;
    if (!ok) return 1e18;
    const double warps = std::min(16, ctas) * std::min(128, ppass * tpm) / 32.0;
    const int cm = cplx ? 4 : 1;
    const double fp_rate = (s.es == 8 && !cplx) || s.es == 16 ? 64.0 : 128.0;
    const double macs = (double)tpm * m.RM * m.RN * K * cm;
    const double t_hbm = pair_bytes / 20.5;
    const double t_smem = c.wf + in_bytes / 128.0;
    const double t_fp = macs / fp_rate;
    const double other = c.ninst + tpm * (60.0 + 3.0 * (m.RM + m.RN) + 7.0 * m.RM * m.RN * (cplx ? 2 : 1)) / 32.0;
    const double eff = std::min(1.0, warps / 8.0) * 0.55;
    const double t_issue = (macs / 32.0 + other) / (4.0 * eff);
    const double t_pipe = t_hbm * (S == 2 ? 1.25 : (S == 3 ? 1.05 : 1.0)) * (ctas < 2 ? 1.5 : 1.0);
    return std::max(std::max(t_pipe, t_smem), std::max(t_fp, t_issue));
}

// Compact search (a few thousand candidates): widest valid vectors, ROTN in
// {0, 1, 2}, S in {2, 3, 4}.  scalar_c: C accessed at arbitrary addresses (VC = 1).
inline Choice search_fast(int es, bool cplx, int M, int N, int K, char opa, char opb, bool b0,
                          bool scalar_c, bool asw = false, bool bsw = false)
{
    Inst s{es, M, N, K, opa, opb, b0};
    s.asw = asw;  // A in the 128-byte-swizzled layout (ASW / ASWG kernels)
    s.bsw = bsw;  // B likewise (BSWG)
    const int wpe = es / 4;
    std::vector<int> rms, rns;
    for (int b = 1; b <= M; ++b) {
        const int r = (M + b - 1) / b;
        if (rms.empty() || rms.back() != r) rms.push_back(r);
    }
    for (int b = 1; b <= N; ++b) {
        const int r = (N + b - 1) / b;
        if (rns.empty() || rns.back() != r) rns.push_back(r);
    }
    Choice best{{std::min(M, 4), std::min(N, 4), 0, 0, 1, 1, 1, 1, 0}, 3, 1e18, 1e18};
    for (int RM : rms)
        for (int RN : rns) {
            if (RM * RN * wpe > 64 || RM > 8 || RN > 16) continue;
            const int tpm = blocks(M, RM) * blocks(N, RN);
            if (tpm > 128) continue;
            const int P = pairs_for(tpm);
            for (int RMODE = 0; RMODE < 2; ++RMODE)
                for (int CMODE = 0; CMODE < 2; ++CMODE)
                    for (int LO = 0; LO < 2; ++LO)
                        for (int ROTN : {0, 1, 2}) {
                            // widest valid vector widths (and scalar C when required)
                            Map m{RM, RN, RMODE, CMODE, LO, 1, 1, 1, ROTN};
                            for (int v : {4, 2}) {
                                Map t = m;
                                t.VA = v;
                                if (valid(s, t)) { m.VA = v; break; }
                            }
                            for (int v : {4, 2}) {
                                Map t = m;
                                t.VB = v;
                                if (valid(s, t)) { m.VB = v; break; }
                            }
                            if (!scalar_c)
                                for (int v : {4, 2}) {
                                    Map t = m;
                                    t.VC = v;
                                    if (valid(s, t)) { m.VC = v; break; }
                                }
                            if (!valid(s, m)) continue;
                            const Cost c = cost(s, m, P);
                            if (c.wf >= 1e8) continue;
                            for (int S = 2; S <= 4; ++S) {
                                int ok = 0;
                                const double pr = predict(s, m, c, S, cplx, ok);
                                if (!ok) continue;
                                const double key = pr + 0.001 * c.wf;
                                if (key < best.pred + 0.001 * best.wf - 1e-9) best = {m, S, pr, c.wf};
                            }
                        }
        }
    return best;
}

}  // namespace txmodel
