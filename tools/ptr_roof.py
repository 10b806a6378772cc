"""Pattern roof of pointer-array batches (measurement tool, not the product).

For each shape and type: the library's pointer-array GEMM and tools/ptr_roof.cu's
plain gather-copy (same bytes, same pointer arrays, no arithmetic) at 10^6 pairs,
pointers in order and randomly permuted.  Prints JSON lines with both times,
the GEMM's fraction of the measured HBM peak and of the pattern's own roof.

  python tools/ptr_roof.py [--shapes 8x16x4,16x3x16,...] [--out file.jsonl]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402
from paper_1304_7053_b200 import model  # noqa: E402

SO = os.path.join(ROOT, "tools", "libptrroof.so")


def lib():
    src = os.path.join(ROOT, "tools", "ptr_roof.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, src])
    L = ctypes.CDLL(SO)
    L.ptr_roof.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_longlong,
                                                                         ctypes.c_void_p,
                                                                         ctypes.c_int,
                                                                         ctypes.c_void_p]
    L.ptr_roof.restype = ctypes.c_int
    return L


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="8x16x4,16x3x16,1x16x16,4x6x16,5x7x3,16x16x1,16x16x16")
    ap.add_argument("--kinds", default="sdcz")
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    L = lib()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = open(a.out, "w") if a.out else None
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for shp in a.shapes.split(","):
        m, n, k = (int(x) for x in shp.split("x"))
        for kind in a.kinds:
            es = model.ESIZE[kind]
            batch = a.batch
            sets = max(1, -(-4 * 126 * 2**20 // (es * (m * k + k * n + m * n) * batch)))
            bufs = []
            for s in range(sets):
                key = lambda nm: txinputs.stream_key(9, "roof", kind, m, n, k, s, nm)
                bufs.append(tuple(txinputs.values_torch(kind, key(nm), 0, e * batch, "cuda")
                                  for nm, e in (("A", m * k), ("B", k * n), ("C", m * n))))
            alpha = txinputs.scalar(kind, 1)
            for order in ("inorder", "permuted"):
                perm = (torch.randperm(batch, generator=torch.Generator().manual_seed(3)).cuda()
                        if order == "permuted" else torch.arange(batch, device="cuda"))
                ptrs = [tuple(x.data_ptr() + perm * (e * es) for x, e in
                              zip(b, (m * k, k * n, m * n))) for b in bufs]
                for general in (False, True):
                    beta = txinputs.scalar(kind, 2) if general else 0
                    it = [0]

                    def gemm():
                        pa, pb, pc = ptrs[it[0] % sets]
                        it[0] += 1
                        rc = tx.tx_gemm_batched_ptr(kind, "N", "N", m, n, k, alpha, pa, m, pb, k,
                                                    beta, pc, m, batch)
                        assert rc == 0, tx.status_string(rc)

                    def roof():
                        pa, pb, pc = ptrs[it[0] % sets]
                        it[0] += 1
                        rc = L.ptr_roof(pa.data_ptr(), pb.data_ptr(), pc.data_ptr(), m * k * es,
                                        k * n * es, m * n * es, 1 if general else 0, batch,
                                        sink.data_ptr(), nsm * 8,
                                        torch.cuda.current_stream().cuda_stream)
                        assert rc == 0

                    byts = model.bytes_moved(kind, m, n, k, batch, True, general)
                    reps = int(max(4, min(100, 10.0 / (byts / (peak * 1e6)))))
                    tg = graph_time(gemm, reps)
                    tr = graph_time(roof, reps)
                    r = {"kind": kind, "m": m, "n": n, "k": k, "order": order, "beta0": not general,
                         "gemm_us": round(tg * 1e3, 2), "roof_us": round(tr * 1e3, 2),
                         "gemm_frac_hbm": round(byts / (tg / 1e3) / 1e9 / peak, 4),
                         "roof_frac_hbm": round(byts / (tr / 1e3) / 1e9 / peak, 4),
                         "gemm_over_roof": round(tr / tg, 4), "sets": sets}
                    print(json.dumps(r), flush=True)
                    if out:
                        out.write(json.dumps(r) + "\n")
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
