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

#include "../paper_1304_7053_b200/csrc/tx_mapmodel.h"
using namespace txmodel;


struct Ty {
    const char *name;
    int es;
    bool cplx;
};

// Best mapping of one square instance under the predicted-time model.
// tra: A is transposed at staging into a padded N-layout copy (ld = n + 1), which
// costs one read and one write of every A element in shared memory plus ~8
// instructions per element (bulk_kernel TRA).
static double search_one(const Ty &t, int n, char pa, char pb, bool b0, bool tra, Map &bestm,
                         Cost &bestc, int &best_S, int qp = 0, bool asw = false, bool pc = false)
{
    pc = pc || asw;  // the power-capped objective (always for ASW instances)
    const int wpe = t.es / 4;
    const int acc_cap = 64;  // accumulator registers per thread
    Inst s{t.es, n, n, n, tra ? 'N' : pa, pb, b0};
    s.asw = asw;  // ASW: P*n <= 256 (TMA box height)
    if (tra) {
        s.ldas = n + 1;
        s.sas = (n + 1) * n + qp;  // qp: extra elements between matrices (bank shift)
    }
    bestc = Cost{1e18, 1e18, 0};
    double best_t = 1e18, best_key = 1e18;
    best_S = 4;
    std::vector<int> rms, rns;
    for (int b = 1; b <= n; ++b) {
        int r = (n + b - 1) / b;
        if (rms.empty() || rms.back() != r) rms.push_back(r);
    }
    rns = rms;
    const int in_bytes = (n * n * 2 + (b0 ? 0 : n * n)) * t.es;
    const int tra_bytes = tra ? ((n + 1) * n + qp) * t.es : 0;  // the padded copy, per pair
    const double pair_bytes = (double)(n * n * (b0 ? 3 : 4)) * t.es;
    const int cm = t.cplx ? 4 : 1;  // real FMAs per complex MAC
    const double fp_rate = t.es == 8 && !t.cplx ? 64.0 : (t.es == 16 ? 64.0 : 128.0);
    const double tra_wf = tra ? 2.0 * n * n * t.es / 128.0 : 0.0;
    const double tra_inst = tra ? 8.0 * n * n / 32.0 : 0.0;
    for (int RM : rms)
        for (int RN : rns) {
            if (RM * RN * wpe > acc_cap) continue;
            const int tpm = blocks(n, RM) * blocks(n, RN);
            if (tpm > 128) continue;
            const int pcap = asw ? 256 / n : 1 << 20;
            const int P = std::min(pairs_for(tpm), pcap);
            for (int S = 2; S <= 4; ++S) {
                // the runtime planner (tx_dispatch.cuh plan_tiles): P = one
                // 128-thread pass x enough passes for a ~16 KB stage
                const int ppass = std::max(1, 128 / tpm);
                const int passes = std::max(1, 16384 / (ppass * in_bytes));
                const long pp = std::min<long>((long)ppass * passes, pcap);
                const long stage = pp * in_bytes;
                const long tra_smem = pp * tra_bytes;
                const int ctas = (int)std::min<long>(16, (225 * 1024L) / (S * stage + tra_smem + 64));
                if (ctas < 2) continue;
                const double warps = ctas * std::min<long>(128, pp * tpm) / 32.0;
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
                                            const double t_smem = c.wf + tra_wf + in_bytes / 128.0;
                                            const double t_fp = macs / fp_rate;
                                            // calibrated on ncu (r01): ~2.2 warp-instructions per
                                            // clock per SM at 8-12 warps; per-item overhead ~40 +
                                            // epilogue ~6 (12 complex) instructions per output
                                            const double other = c.ninst + tra_inst + tpm * (60.0 + 3.0 * (RM + RN) + 7.0 * RM * RN * (t.cplx ? 2 : 1)) / 32.0;
                                            const double eff = std::min(1.0, warps / 8.0) * 0.55;
                                            const double t_issue = (macs / 32.0 + other) / (4.0 * eff);
                                            // fewer stages than 3 exposes DRAM latency between tiles
                                            const double t_pipe = t_hbm * (S == 2 ? 1.25 : (S == 3 ? 1.05 : 1.0));
                                            const double t_sm = std::max(t_smem, std::max(t_fp, t_issue));
                                            const double tp = std::max(t_pipe, t_sm);
                                            // pc: the SM-side time at a power-capped clock (~0.7 x
                                            // max, as sustained runs see) against the HBM time
                                            const double key = pc ? std::max(t_sm / 0.7, t_pipe) + 0.01 * t_sm + 0.0001 * c.regs
                                                                   : tp + 0.001 * c.wf + 0.0001 * c.regs;
                                            if (key < best_key - 1e-9) {
                                                best_key = key;
                                                best_t = tp;
                                                bestc = c;
                                                bestm = m;
                                                best_S = S;
                                            }
                                        }
            }
        }
    return best_t;
}

// usage: mapsearch [n]           -> tx_map_table.inc candidates (every square instance)
//        mapsearch --tra TABLE   -> TX_TRAMAP lines for the instances TABLE marks TRA
int main(int argc, char **argv)
{
    Ty types[] = {{"float", 4, false}, {"double", 8, false}, {"float2", 8, true}, {"double2", 16, true}};
    if (argc > 2 && std::strcmp(argv[1], "--tra") == 0) {
        FILE *f = std::fopen(argv[2], "r");
        if (!f) return 1;
        char line[512];
        printf("// Generated by tools/mapsearch.cpp --tra -- do not edit.  Compute mapping of the\n");
        printf("// TRA instances (A transposed at staging into a padded N-layout copy, ld = n + 1).\n");
        printf("// TX_TRAMAP(T, n, OPA, OPB, B0, RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN, S, ON)\n");
        printf("// ON: set by measurement (tools/merge_tra.py)\n");
        while (std::fgets(line, sizeof line, f)) {
            char tn[16];
            int v[16];
            if (std::sscanf(line, "TX_MAP(%15[^,], %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d)",
                            tn, &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6], &v[7], &v[8], &v[9],
                            &v[10], &v[11], &v[12], &v[13], &v[14], &v[15]) != 17)
                continue;
            if (!v[15] || v[1] == 0) continue;  // not a TRA instance
            const Ty *t = nullptr;
            for (auto &x : types)
                if (std::strcmp(x.name, tn) == 0) t = &x;
            if (!t) continue;
            const int n = v[0];
            Map bm{};
            Cost bc{};
            int bS = 0, bq = 0;
            double pt = 1e18;
            for (int qp : {0}) {  // the kernel's padded copy has no per-matrix pad (QP = 0)
                Map m{};
                Cost c{};
                int S = 0;
                const double p = search_one(*t, n, 'T', v[2] == 0 ? 'N' : 'T', v[3] != 0, true, m, c, S, qp);
                if (p + 0.001 * c.wf < pt + 0.001 * bc.wf - 1e-9) {
                    pt = p;
                    bm = m;
                    bc = c;
                    bS = S;
                    bq = qp;
                }
            }
            (void)bq;
            printf("TX_TRAMAP(%s, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, 1) "
                   "// wf %.1f inst %.1f regs %d pred %.0f clk/pair (own entry RM %d RN %d)\n",
                   t->name, n, v[1], v[2], v[3], bm.RM, bm.RN, bm.RMODE, bm.CMODE, bm.LO, bm.VA,
                   bm.VB, bm.VC, bm.ROTN, bS, bc.wf, bc.ninst, bc.regs, pt, v[4], v[5]);
        }
        std::fclose(f);
        return 0;
    }
    if (argc > 1 && std::strcmp(argv[1], "--asw") == 0) {
        // ASW candidates: n = 16 with 8- and 16-byte elements (a stored row is 128 or
        // 256 bytes), op(A) = T/C, every op(B), beta == 0 and general.  The last column
        // (ON) is set by measurement (tools/apply_asw.py).
        printf("// Generated by tools/mapsearch.cpp --asw; ON column set by measurement.\n");
        printf("// TX_ASWMAP(T, n, OPA, OPB, B0, RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN, S, KB, ON)\n");
        const int n = 16;
        for (auto &t : types) {
            if (t.es < 8) continue;
            const char *ops = t.cplx ? "NTC" : "NT";
            for (const char *pa = ops + 1; *pa; ++pa)
                for (const char *pb = ops; *pb; ++pb)
                    for (int b0 = 0; b0 < 2; ++b0) {
                        Map bm{};
                        Cost bc{};
                        int bS = 0;
                        const double pt = search_one(t, n, 'T', *pb == 'N' ? 'N' : 'T', b0 == 1, false,
                                                     bm, bc, bS, 0, true);
                        const int opa = *pa == 'T' ? 1 : 2;
                        const int opb = *pb == 'N' ? 0 : (*pb == 'T' ? 1 : 2);
                        printf("TX_ASWMAP(%s, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, 16, 1) "
                               "// wf %.1f inst %.1f regs %d pred %.0f clk/pair\n",
                               t.name, n, opa, opb, b0, bm.RM, bm.RN, bm.RMODE, bm.CMODE, bm.LO, bm.VA,
                               bm.VB, bm.VC, bm.ROTN, bS, bc.wf, bc.ninst, bc.regs, pt);
                        fflush(stdout);
                    }
        }
        return 0;
    }
    if (argc > 4 && std::strcmp(argv[1], "--pc") == 0) {
        // re-search square instances of the given types (e.g. "zc") and sizes with the
        // power-capped objective; TX_MAP lines with S from the search and 16 KB stages
        const char *kinds = argv[2];
        const int lo = atoi(argv[3]), hi = atoi(argv[4]);
        for (auto &t : types) {
            const char tk = t.es == 4 ? 's' : (t.es == 8 ? (t.cplx ? 'c' : 'd') : 'z');
            if (!std::strchr(kinds, tk)) continue;
            for (int n = lo; n <= hi; ++n) {
                const char *ops = t.cplx ? "NTC" : "NT";
                for (const char *pa = ops; *pa; ++pa)
                    for (const char *pb = ops; *pb; ++pb)
                        for (int b0 = 0; b0 < 2; ++b0) {
                            const char ca = *pa == 'N' ? 'N' : 'T', cb = *pb == 'N' ? 'N' : 'T';
                            Map bm{};
                            Cost bc{};
                            int bS = 0;
                            const double pt = search_one(t, n, ca, cb, b0 == 1, false, bm, bc, bS, 0,
                                                         false, true);
                            const int opa = *pa == 'N' ? 0 : (*pa == 'T' ? 1 : 2);
                            const int opb = *pb == 'N' ? 0 : (*pb == 'T' ? 1 : 2);
                            printf("TX_MAP(%s, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, %d, 16, 0) "
                                   "// pc search: wf %.1f inst %.1f regs %d pred %.0f clk/pair\n",
                                   t.name, n, opa, opb, b0, bm.RM, bm.RN, bm.RMODE, bm.CMODE, bm.LO,
                                   bm.VA, bm.VB, bm.VC, bm.ROTN, bS, bc.wf, bc.ninst, bc.regs, pt);
                            fflush(stdout);
                        }
            }
        }
        return 0;
    }
    int only_n = argc > 1 ? atoi(argv[1]) : 0;
    printf("// Generated by tools/mapsearch.cpp -- do not edit.  Columns:\n");
    printf("// TX_MAP(T, n, OPA, OPB, B0, RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN, S)\n");
    for (auto &t : types) {
        for (int n = 1; n <= 16; ++n) {
            if (only_n && n != only_n) continue;
            const char *ops = t.cplx ? "NTC" : "NT";
            for (const char *pa = ops; *pa; ++pa)
                for (const char *pb = ops; *pb; ++pb)
                    for (int b0 = 0; b0 < 2; ++b0) {
                        const char ca = *pa == 'N' ? 'N' : 'T', cb = *pb == 'N' ? 'N' : 'T';
                        Inst s{t.es, n, n, n, ca, cb, b0 == 1};
                        Map bestm{};
                        Cost bestc{};
                        int best_S = 0;
                        const double best_t = search_one(t, n, ca, cb, b0 == 1, false, bestm, bestc, best_S);
                        int r4 = std::min(4, n);
                        int r4b = blocks(n, blocks(n, r4));
                        Map base{r4b, r4b, 0, 0, 1, 1, 1, 1, 0};
                        Cost bc = cost(s, base, pairs_for(blocks(n, r4b) * blocks(n, r4b)));
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
