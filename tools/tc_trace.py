"""Timeline of the tensor-core kernel's CTA 0 (tools/tc_trace.cu; needs a GPU).

  python tools/tc_trace.py c 32 32 32 gen [batch] [--so lib.so] [--quiet]

Variants of the kernel for experiments: build tools/tc_trace.cu with -D flags into another
.so and pass --so.  Also prints the launch's device time and its fraction of the HBM peak.

Prints, per operand unit / pair, cycles (clock64, relative to the first producer issue) of:
producer tile issue (P), transform start / end (T0/T1), MMA start / committed (M0/M1),
epilogue start / end (E0/E1), and the steady-state cycles per pair."""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "libtctrace.so")


def main():
    argv = [a for a in sys.argv[1:]]
    so = SO
    if "--so" in argv:
        i = argv.index("--so")
        so = argv[i + 1]
        del argv[i:i + 2]
    quiet = "--quiet" in argv
    argv = [a for a in argv if a != "--quiet"]
    kind, m, n, k, b = argv[0], int(argv[1]), int(argv[2]), int(argv[3]), argv[4]
    batch = int(argv[5]) if len(argv) > 5 else 100000
    src = os.path.join(ROOT, "tools", "tc_trace.cu")
    deps = [src, os.path.join(ROOT, "paper_1304_7053_b200", "csrc", "tx_tc.cuh")]
    if so == SO and (not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(d) for d in deps)):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I",
                               os.path.join(ROOT, "paper_1304_7053_b200", "csrc"), "-shared", "-Xcompiler",
                               "-fPIC", "-o", SO, src])
    import torch

    L = ctypes.CDLL(so)
    cplx = kind == "c"
    es = 8 if cplx else 4
    A = torch.rand(batch * m * k * es // 4, device="cuda")
    B = torch.rand(batch * k * n * es // 4, device="cuda")
    C = torch.rand(batch * m * n * es // 4, device="cuda")
    out = np.zeros((8, 256), dtype=np.uint64)
    ms = ctypes.c_float(0)
    times = []
    for rep in range(5):
        rc = L.tc_trace_run(int(cplx), int(b == "b0"), m, n, k, batch, ctypes.c_void_p(A.data_ptr()),
                            ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(ms))
        assert rc == 0, rc
        times.append(ms.value)
    byts = batch * es * (m * k + k * n + m * n * (1 if b == "b0" else 2))
    best = min(times[1:])
    print(f"{kind}{m}x{n}x{k} {b} batch={batch}: {best * 1e3:.1f} us, {byts / best / 1e6:.0f} GB/s, "
          f"{byts / best / 1e6 / 6446.9:.3f} of measured HBM ({os.path.basename(so)})")
    if quiet:
        return
    t0 = int(out[0][0])
    rel = lambda v: int(v) - t0 if v else -1
    names = ["P", "T0", "T1", "M0", "M1", "E0", "E1"]
    print(" idx " + " ".join(f"{x:>8}" for x in names))
    for i in range(40):
        print(f"{i:4d} " + " ".join(f"{rel(out[e][i]):8d}" for e in range(7)))
    e1 = [int(v) for v in out[6][:200] if v]
    if len(e1) > 60:
        print("steady cycles/pair (epilogue end, pairs 20..60):", (e1[60] - e1[20]) / 40)


if __name__ == "__main__":
    main()
