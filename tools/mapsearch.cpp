// mapsearch.cpp -- offline search of the per-instance compute mapping of the
// size-specialised bulk kernels (same model as tools/mapsim.py, in C++ so the
// whole space can be enumerated).  Emits paper_1304_7053_b200/csrc/tx_map_table.inc.
//
// A mapping assigns thread (matrix q of the tile, row block rb, column block cb)
// an RM x RN micro-tile; RMODE/CMODE choose blocked or interleaved rows/cols,
// ROTN rotates a thread's columns by q*ROTN (mod N), LO picks which of rb/cb is
// the fastest-varying lane index, VA/VB/VC are the vector widths (elements) of
// the A/B/C shared-memory accesses.  Every mapping keeps each output's sum in
// ascending l, so all mappings give bitwise-identical results.
//
// Cost model: per warp instruction, lanes form phases of 128/bytes lanes; a
// phase costs the max over the 32 banks of the distinct 4-byte words it
// requests.  Score = wavefronts per pair (compute loads + C in) + 128-byte
// lines touched by the global C stores,
// ties broken by instructions per pair, then registers.
//
//   g++ -O2 -std=c++17 -o /tmp/mapsearch tools/mapsearch.cpp && /tmp/mapsearch > ...
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

struct Map {
    int RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN;
};

static int blocks(int n, int r) { return (n + r - 1) / r; }

static int wavefronts(const long *addr, int nwords, const bool *act)
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
};

static bool valid(const Inst &s, const Map &m)
{
    const int SA = s.M * s.K, SB = s.K * s.N, SC = s.M * s.N;
    for (int v : {m.VA, m.VB, m.VC})
        if (v * s.es > 16) return false;
    const int RB = blocks(s.M, m.RM), CB = blocks(s.N, m.RN);
    if (m.RM * RB - s.M >= m.RM || m.RN * CB - s.N >= m.RN) return false;
    if (m.VA > 1) {
        if (SA % m.VA) return false;
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

static Cost cost(const Inst &s, const Map &m, int P)
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
                        for (int ln = 0; ln < 32; ++ln)
                            addr[ln] = (A0 + (long)q[ln] * SA + row(ln, g) + (long)M * l) * wpe;
                        wf += wavefronts(addr, v * wpe, act);
                        ++ni;
                    }
            } else {
                const int v = VLa;
                for (int r = 0; r < m.RM; ++r)
                    for (int l = l0; l < l0 + VL; l += v) {
                        for (int ln = 0; ln < 32; ++ln)
                            addr[ln] = (A0 + (long)q[ln] * SA + l + (long)K * row(ln, r)) * wpe;
                        wf += wavefronts(addr, v * wpe, act);
                        ++ni;
                    }
            }
            // B
            if (s.opb == 'N') {
                const int v = VLb;
                for (int cc = 0; cc < m.RN; ++cc)
                    for (int l = l0; l < l0 + VL; l += v) {
                        for (int ln = 0; ln < 32; ++ln)
                            addr[ln] = (B0 + (long)q[ln] * SB + l + (long)K * col(ln, cc)) * wpe;
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

static int pairs_for(const Inst &s, int tpm)
{
    const int NT = 128;
    int ppass = std::max(1, NT / tpm);
    // simulate ~8 warps worth of items, at least one full pass
    int P = std::max(ppass, (8 * 32 + tpm - 1) / tpm);
    return P;
}

int main(int argc, char **argv)
{
    struct T {
        const char *name;
        int es;
        bool cplx;
    } types[] = {{"float", 4, false}, {"double", 8, false}, {"float2", 8, true}, {"double2", 16, true}};
    int only_n = argc > 1 ? atoi(argv[1]) : 0;
    printf("// Generated by tools/mapsearch.cpp -- do not edit.  Columns:\n");
    printf("// TX_MAP(T, n, OPA, OPB, B0, RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN, S)\n");
    for (auto &t : types) {
        const int wpe = t.es / 4;
        const int acc_cap = 64;  // accumulator registers per thread
        for (int n = 1; n <= 16; ++n) {
            if (only_n && n != only_n) continue;
            const char *ops = t.cplx ? "NTC" : "NT";
            for (const char *pa = ops; *pa; ++pa)
                for (const char *pb = ops; *pb; ++pb)
                    for (int b0 = 0; b0 < 2; ++b0) {
                        Inst s{t.es, n, n, n, *pa == 'N' ? 'N' : 'T', *pb == 'N' ? 'N' : 'T', b0 == 1};
                        Map bestm{};
                        Cost bestc{1e18, 1e18, 0};
                        double best_t = 1e18;
                        int best_S = 4;
                        std::vector<int> rms, rns;
                        for (int b = 1; b <= n; ++b) {
                            int r = (n + b - 1) / b;
                            if (rms.empty() || rms.back() != r) rms.push_back(r);
                        }
                        rns = rms;
                        const int in_bytes = (n * n * 2 + (b0 ? 0 : n * n)) * t.es;
                        const double pair_bytes = (double)(n * n * (b0 ? 3 : 4)) * t.es;
                        const int cm = t.cplx ? 4 : 1;          // real FMAs per complex MAC
                        const double fp_rate = t.es == 8 && !t.cplx ? 64.0 : (t.es == 16 ? 64.0 : 128.0);
                        for (int RM : rms)
                            for (int RN : rns) {
                                if (RM * RN * wpe > acc_cap) continue;
                                const int tpm = blocks(n, RM) * blocks(n, RN);
                                if (tpm > 128) continue;
                                const int P = pairs_for(s, tpm);
                                for (int S = 2; S <= 4; ++S) {
                                    // the runtime planner (tx_dispatch.cuh plan_tiles): P = one
                                    // 128-thread pass x enough passes for a ~16 KB stage
                                    const int ppass = std::max(1, 128 / tpm);
                                    const int passes = std::max(1, 16384 / (ppass * in_bytes));
                                    const long stage = (long)ppass * passes * in_bytes;
                                    const int ctas = (int)std::min<long>(16, (225 * 1024L) / (S * stage + 64));
                                    if (ctas < 2) continue;
                                    const double warps = ctas * std::min(128, ppass * tpm) / 32.0;
                                    for (int RMODE = 0; RMODE < 2; ++RMODE)
                                        for (int CMODE = 0; CMODE < 2; ++CMODE)
                                            for (int LO = 0; LO < 2; ++LO)
                                                for (int VA : {1, 2, 4})
                                                    for (int VB : {1, 2, 4})
                                                        for (int VC : {1, 2, 4})
                                                            for (int ROTN : {0, 1, 2, 3, 4}) {
                                                                Map m{RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN};
                                                                if (!valid(s, m)) continue;
                                                                Cost c = cost(s, m, P);
                                                                // ---- predicted cycles per pair per SM
                                                                const double macs = (double)tpm * RM * RN * n * cm;
                                                                const double t_hbm = pair_bytes / 20.5;
                                                                const double t_smem = c.wf + in_bytes / 128.0;
                                                                const double t_fp = macs / fp_rate;
                                                                // calibrated on ncu (r01): ~2.2 warp-instructions per
                                                                // clock per SM at 8-12 warps; per-item overhead ~40 +
                                                                // epilogue ~6 (12 complex) instructions per output
                                                                const double other = c.ninst + tpm * (60.0 + 3.0 * (RM + RN) + 7.0 * RM * RN * (t.cplx ? 2 : 1)) / 32.0;
                                                                const double eff = std::min(1.0, warps / 8.0) * 0.55;
                                                                const double t_issue = (macs / 32.0 + other) / (4.0 * eff);
                                                                // fewer stages than 3 exposes DRAM latency between tiles
                                                                const double t_pipe = t_hbm * (S == 2 ? 1.25 : (S == 3 ? 1.05 : 1.0));
                                                                const double tp = std::max(std::max(t_pipe, t_smem), std::max(t_fp, t_issue));
                                                                const double key = tp + 0.001 * c.wf + 0.0001 * c.regs;
                                                                if (key < best_t - 1e-9) {
                                                                    best_t = key;
                                                                    bestc = c;
                                                                    bestm = m;
                                                                    best_S = S;
                                                                }
                                                            }
                                }
                            }
                        int r4 = std::min(4, n);
                        int r4b = blocks(n, blocks(n, r4));
                        Map base{r4b, r4b, 0, 0, 1, 1, 1, 1, 0};
                        Cost bc = cost(s, base, pairs_for(s, blocks(n, r4b) * blocks(n, r4b)));
                        int opa = *pa == 'N' ? 0 : (*pa == 'T' ? 1 : 2);
                        int opb = *pb == 'N' ? 0 : (*pb == 'T' ? 1 : 2);
                        printf("TX_MAP(%s, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d) "
                               "// wf %.1f inst %.1f regs %d pred %.0f clk/pair hbm %.0f (base wf %.1f)\n",
                               t.name, n, opa, opb, b0, bestm.RM, bestm.RN, bestm.RMODE,
                               bestm.CMODE, bestm.LO, bestm.VA, bestm.VB, bestm.VC, bestm.ROTN,
                               best_S, bestc.wf, bestc.ninst, bestc.regs, best_t,
                               (double)(n * n * (b0 ? 3 : 4)) * t.es / 20.5, bc.wf);
                        fflush(stdout);
                    }
        }
    }
    return 0;
}
