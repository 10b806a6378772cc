"""Shared-memory bank-conflict simulator for the compute mapping of the batched
GEMM kernels (paper_1304_7053_b200/csrc/tx_kernels.cuh).

A mapping assigns each thread of a CTA one work item (matrix q of the tile,
row block rb, column block cb) and fixes how its RM x RN micro-tile reads the
packed shared-memory stage:

  rows  i_r = rb*RM + r (RMODE 0, blocked)  or rb + RB*r (RMODE 1, interleaved)
  cols  j_c = cb*RN + c (CMODE 0)           or cb + CB*c (CMODE 1),
        then rotated per matrix: (j_c + q*ROTN) mod N  (ROTN; keeps every output's
        sum in ascending l, only WHICH columns a thread owns changes)
  lanes sub = rb + RB*cb (LO 0, rb fastest) or cb + CB*rb (LO 1)
  VA / VB / VC: vector width (elements) of the A / B / C shared-memory accesses
        along the stored-contiguous dimension (A-N: rows, A-T: l, B-N: l,
        B-T: cols, C: rows).

Wavefront model (per warp instruction): lanes are split into phases of
128/access_bytes lanes; a phase costs max over the 32 four-byte banks of the
number of DISTINCT words requested in that bank (broadcast is free).

`best(...)` enumerates mappings and returns the one with the fewest wavefronts
per pair (ties: fewer LDS instructions, fewer registers).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np

NT = 128


@dataclass(frozen=True)
class Mapping:
    RM: int
    RN: int
    RMODE: int
    CMODE: int
    LO: int
    VA: int
    VB: int
    VC: int
    ROTN: int


def blocks(n, r):
    return (n + r - 1) // r


def phase_wavefronts(addr_words, nwords, active):
    """addr_words: (32,) first 4-byte word of each lane's access; nwords = words per
    access (1, 2 or 4); active: (32,) bool.  Returns wavefronts of one instruction."""
    lanes_per_phase = 32 // nwords
    total = 0
    for p0 in range(0, 32, lanes_per_phase):
        sl = slice(p0, p0 + lanes_per_phase)
        a = addr_words[sl][active[sl]]
        if a.size == 0:
            continue
        words = np.unique((a[:, None] + np.arange(nwords)[None, :]).ravel())
        banks = words % 32
        total += int(np.bincount(banks, minlength=32).max())
    return total


class Sim:
    def __init__(self, es, M, N, K, opa, opb, b0, P):
        self.es, self.M, self.N, self.K = es, M, N, K
        self.opa, self.opb, self.b0, self.P = opa, opb, b0, P
        self.wpe = es // 4  # 4-byte words per element
        self.SA, self.SB, self.SC = M * K, K * N, M * N

    def valid(self, mp: Mapping):
        M, N, K, es = self.M, self.N, self.K, self.es
        for v in (mp.VA, mp.VB, mp.VC):
            if v * es > 16:
                return False
        RB, CB = blocks(M, mp.RM), blocks(N, mp.RN)
        if mp.RM * RB - M >= mp.RM or mp.RN * CB - N >= mp.RN:
            return False
        # A vector
        if mp.VA > 1:
            if self.SA % mp.VA:
                return False
            if self.opa == "N":
                if mp.RMODE != 0 or mp.RM % mp.VA or M % mp.VA:
                    return False
            else:
                if K % mp.VA:
                    return False
        if mp.VB > 1:
            if self.SB % mp.VB:
                return False
            if self.opb == "N":
                if K % mp.VB:
                    return False
            else:
                if mp.CMODE != 0 or mp.RN % mp.VB or N % mp.VB or mp.ROTN % mp.VB:
                    return False
        if mp.VC > 1:
            if mp.RMODE != 0 or mp.RM % mp.VC or M % mp.VC or self.SC % mp.VC:
                return False
        if mp.ROTN and mp.CMODE == 0 and mp.VB > 1 and self.opb != "N":
            pass
        return True

    def lanes(self, mp: Mapping, warp):
        RB, CB = blocks(self.M, mp.RM), blocks(self.N, mp.RN)
        tpm = RB * CB
        w = warp * 32 + np.arange(32)
        active = w < self.P * tpm
        q = w // tpm
        sub = w % tpm
        if mp.LO == 0:
            rb, cb = sub % RB, sub // RB
        else:
            cb, rb = sub % CB, sub // CB
        return q, rb, cb, active, RB, CB

    def rows(self, mp, rb, RB, r):
        i = rb * mp.RM + r if mp.RMODE == 0 else rb + RB * r
        return np.minimum(i, self.M - 1)

    def cols(self, mp, cb, CB, c, q):
        j = cb * mp.RN + c if mp.CMODE == 0 else cb + CB * c
        j = np.minimum(j, self.N - 1)
        if mp.ROTN:
            j = (j + q * mp.ROTN) % self.N
        return j

    def cost(self, mp: Mapping):
        """(wavefronts per pair, LDS+STS instructions per pair)."""
        M, N, K, wpe = self.M, self.N, self.K, self.wpe
        RB, CB = blocks(M, mp.RM), blocks(N, mp.RN)
        tpm = RB * CB
        items = self.P * tpm
        nwarps = (items + 31) // 32
        VLa = mp.VA if (self.opa != "N" and mp.VA > 1) else 1
        VLb = mp.VB if (self.opb == "N" and mp.VB > 1) else 1
        VL = max(VLa, VLb)
        if K % VL:
            return None
        wf = 0
        ninst = 0
        A0, B0, C0 = 0, self.P * self.SA, self.P * (self.SA + self.SB)
        for wi in range(nwarps):
            q, rb, cb, act, _, _ = self.lanes(mp, wi)
            for l0 in range(0, K, VL):
                # ---- A loads
                if self.opa == "N":
                    if mp.VA > 1:
                        for g in range(mp.RM // mp.VA):
                            i = self.rows(mp, rb, RB, g * mp.VA)
                            for l in range(l0, l0 + VL):
                                a = (A0 + q * self.SA + i + M * l) * wpe
                                wf += phase_wavefronts(a, mp.VA * wpe, act)
                                ninst += 1
                    else:
                        for r in range(mp.RM):
                            i = self.rows(mp, rb, RB, r)
                            for l in range(l0, l0 + VL):
                                a = (A0 + q * self.SA + i + M * l) * wpe
                                wf += phase_wavefronts(a, wpe, act)
                                ninst += 1
                else:
                    for r in range(mp.RM):
                        i = self.rows(mp, rb, RB, r)
                        step = mp.VA if mp.VA > 1 else 1
                        for l in range(l0, l0 + VL, step):
                            a = (A0 + q * self.SA + l + K * i) * wpe
                            wf += phase_wavefronts(a, step * wpe, act)
                            ninst += 1
                # ---- B loads
                if self.opb == "N":
                    for c in range(mp.RN):
                        j = self.cols(mp, cb, CB, c, q)
                        step = mp.VB if mp.VB > 1 else 1
                        for l in range(l0, l0 + VL, step):
                            a = (B0 + q * self.SB + l + K * j) * wpe
                            wf += phase_wavefronts(a, step * wpe, act)
                            ninst += 1
                else:
                    if mp.VB > 1:
                        for g in range(mp.RN // mp.VB):
                            j = self.cols(mp, cb, CB, g * mp.VB, q)
                            for l in range(l0, l0 + VL):
                                a = (B0 + q * self.SB + j + N * l) * wpe
                                wf += phase_wavefronts(a, mp.VB * wpe, act)
                                ninst += 1
                    else:
                        for c in range(mp.RN):
                            j = self.cols(mp, cb, CB, c, q)
                            for l in range(l0, l0 + VL):
                                a = (B0 + q * self.SB + j + N * l) * wpe
                                wf += phase_wavefronts(a, wpe, act)
                                ninst += 1
            # ---- epilogue: C in (beta != 0) and out tile
            for c in range(mp.RN):
                j = self.cols(mp, cb, CB, c, q)
                step = mp.VC if mp.VC > 1 else 1
                for r in range(0, mp.RM, step):
                    i = self.rows(mp, rb, RB, r)
                    a_in = (C0 + q * self.SC + i + M * j) * wpe
                    a_out = (q * self.SC + i + M * j) * wpe  # separate out buffer
                    reps = 1 if self.b0 else 2
                    for a in ([a_out] if self.b0 else [a_in, a_out]):
                        wf += phase_wavefronts(a, step * wpe, act)
                        ninst += 1
        return wf / self.P, ninst / self.P

    def regs(self, mp):
        R = self.wpe
        VLa = mp.VA if (self.opa != "N" and mp.VA > 1) else 1
        VLb = mp.VB if (self.opb == "N" and mp.VB > 1) else 1
        VL = max(VLa, VLb)
        return mp.RM * mp.RN * R + (mp.RM + mp.RN) * VL * R + 24


def tile_pairs(es, M, N, K, b0, tpm):
    """Pairs per tile the host planner would use (16 KB stage target)."""
    SA, SB, SC = M * K, K * N, M * N
    inb = (SA + SB + (0 if b0 else SC)) * es
    align = 16 // math.gcd(16, math.gcd(SA * es, math.gcd(SB * es, SC * es)))
    ppass = max(1, NT // tpm)
    passes = max(1, 16384 // (ppass * inb))
    P = ppass * passes
    P = ((P + align - 1) // align) * align
    return P


def candidates(es, M, N, K, opa, opb, acc_cap):
    R = es // 4
    rms = sorted({blocks(M, rb) and -(-M // rb) for rb in range(1, M + 1)})
    rns = sorted({-(-N // cb) for cb in range(1, N + 1)})
    for RM in rms:
        for RN in rns:
            if RM * RN * R > acc_cap:
                continue
            if RM * RN * R < min(8, M * N * R):
                continue
            tpm = blocks(M, RM) * blocks(N, RN)
            if tpm > NT:
                continue
            for RMODE, CMODE, LO in itertools.product((0, 1), (0, 1), (0, 1)):
                for VA in (1, 2, 4):
                    for VB in (1, 2, 4):
                        for VC in (1, 2, 4):
                            for ROTN in (0, 1, 2, 4):
                                if ROTN >= N:
                                    continue
                                yield Mapping(RM, RN, RMODE, CMODE, LO, VA, VB, VC, ROTN)


def best(es, M, N, K, opa, opb, b0, acc_cap=None, top=1, verbose=False):
    R = es // 4
    if acc_cap is None:
        acc_cap = 64
    results = []
    sims = {}
    for mp in candidates(es, M, N, K, opa, opb, acc_cap):
        tpm = blocks(M, mp.RM) * blocks(N, mp.RN)
        P = tile_pairs(es, M, N, K, b0, tpm)
        P = min(P, max(1, 4 * 32 // math.gcd(32, tpm)) * 4)  # simulate a few warps only
        key = P
        if key not in sims:
            sims[key] = Sim(es, M, N, K, opa, opb, b0, P)
        s = sims[key]
        if not s.valid(mp):
            continue
        c = s.cost(mp)
        if c is None:
            continue
        wf, ni = c
        results.append((wf, ni, s.regs(mp), mp))
    results.sort(key=lambda t: (round(t[0], 3), t[1], t[2]))
    if verbose:
        for r in results[:top]:
            print(r)
    return results[:top]


def ideal(es, M, N, K):
    """Lower bound on compute-read wavefronts per pair for a 4x4-ish tile."""
    return None


if __name__ == "__main__":
    import sys
    import time

    es, n, opa, opb, b0 = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5] == "1"
    t = time.time()
    best(es, n, n, n, opa, opb, b0, top=8, verbose=True)
    print("default 4x4:", Sim(es, n, n, n, opa, opb, b0, 16).cost(Mapping(min(4, n), min(4, n), 0, 0, 1, 1, 1, 1, 0)))
    print(f"{time.time() - t:.1f}s")
