"""What the FP64 tensor-core MMA computes (measurement tool): compare D = A*B + C
from mma.sync m8n8k4 f64 with candidate evaluation orders, bit for bit.

  python tools/dmma_probe.py        (needs a GPU; builds tools/libdmmaprobe.so)
"""
import ctypes
import json
import math
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "libdmmaprobe.so")


def fma(a, b, c):
    """Correctly rounded a*b + c via exact rationals."""
    from fractions import Fraction

    return float(Fraction(a) * Fraction(b) + Fraction(c))


def main():
    src = os.path.join(ROOT, "tools", "dmma_probe.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, src])
    import torch

    L = ctypes.CDLL(SO)
    nw = 256
    rng = np.random.default_rng(1)
    res = {}
    for dist in ("uniform", "wide"):
        if dist == "uniform":
            A = rng.uniform(-1, 1, (nw, 8, 4))
            B = rng.uniform(-1, 1, (nw, 4, 8))
            C = rng.uniform(-1, 1, (nw, 8, 8))
        else:  # magnitudes spread over 2^-30..2^30: exposes the alignment / rounding policy
            A = rng.uniform(-1, 1, (nw, 8, 4)) * 2.0 ** rng.integers(-30, 30, (nw, 8, 4))
            B = rng.uniform(-1, 1, (nw, 4, 8)) * 2.0 ** rng.integers(-30, 30, (nw, 4, 8))
            C = rng.uniform(-1, 1, (nw, 8, 8)) * 2.0 ** rng.integers(-30, 30, (nw, 8, 8))
        dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, C))
        dD = torch.empty_like(dC)
        assert L.dmma_probe(ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                            ctypes.c_void_p(dC.data_ptr()), ctypes.c_void_p(dD.data_ptr()),
                            nw) == 0
        D = dD.cpu().numpy()
        counts = {"seq_k0_first": 0, "seq_k3_first": 0, "exact_rounded_once": 0,
                  "products_tree": 0, "none": 0, "total": 0}
        from fractions import Fraction
        worst_ulp = 0.0
        for w in range(nw):
            for i in range(8):
                for j in range(8):
                    a, b, c, d = A[w, i], B[w, :, j], C[w, i, j], D[w, i, j]
                    s = c
                    for k in range(4):
                        s = fma(a[k], b[k], s)
                    r = c
                    for k in (3, 2, 1, 0):
                        r = fma(a[k], b[k], r)
                    ex = float(Fraction(c) + sum(Fraction(a[k]) * Fraction(b[k]) for k in range(4)))
                    p = [float(Fraction(a[k]) * Fraction(b[k])) for k in range(4)]
                    tree = (p[0] + p[1]) + (p[2] + p[3]) + c
                    counts["total"] += 1
                    hit = False
                    if d == s:
                        counts["seq_k0_first"] += 1
                        hit = True
                    if d == r:
                        counts["seq_k3_first"] += 1
                        hit = True
                    if d == ex:
                        counts["exact_rounded_once"] += 1
                        hit = True
                    if d == tree:
                        counts["products_tree"] += 1
                        hit = True
                    if not hit:
                        counts["none"] += 1
                    if ex != 0:
                        worst_ulp = max(worst_ulp, abs(d - ex) / math.ulp(ex))
        counts["worst_ulp_vs_exact"] = worst_ulp
        res[dist] = counts
    L.dmma_rate.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
    L.dmma_rate.restype = ctypes.c_float
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for which, name in ((0, "dmma"), (1, "dfma")):
        for threads in (128, 256, 512):
            blocks, iters = nsm * 4, 2000
            ms = L.dmma_rate(which, blocks, threads, iters, out.data_ptr())
            if which == 0:
                flops = blocks * (threads // 32) * iters * 8 * (8 * 8 * 4 * 2)
            else:
                flops = blocks * threads * iters * 32 * 8 * 2
            res[f"{name}_tflops_{threads}thr"] = round(flops / (ms / 1e3) / 1e12, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
