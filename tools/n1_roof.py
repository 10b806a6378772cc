"""Size-matched streaming roof for n = 1, 2 (measurement tool, not the product).

At n = 1 a batched GEMM is an elementwise product: C = alpha*A*B (+ beta*C).  PyTorch's own
elementwise kernels over the same tensors move exactly the same bytes (A, B read, C read
when beta != 0, C written), so their time under the gate protocol (CUDA graph of back-to-back
calls over rotating sets >= 4 x L2, 10^6 pairs) is the practical roof of a call this small
(launch ramp + one DRAM round trip + drain dominate a 12-48 MB call).  For n = 2 the same
elementwise kernels over the same byte counts serve as the roof.  Prints one JSON line per
(kind, n, beta) with both times and fractions of the measured HBM peak.

  python tools/n1_roof.py [--out file.jsonl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402
from paper_1304_7053_b200 import model  # noqa: E402


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
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = open(a.out, "w") if a.out else None
    batch = a.batch
    for kind in "sdcz":
        for n in (1, 2):
            e = n * n
            es = model.ESIZE[kind]
            sets = max(1, -(-4 * 126 * 2**20 // (es * 3 * e * batch)))
            bufs = [tuple(txinputs.values_torch(kind, txinputs.stream_key(5, "n1", kind, n, s, nm),
                                                0, e * batch, "cuda") for nm in "ABC")
                    for s in range(sets)]
            alpha = txinputs.scalar(kind, 1)
            for general in (False, True):
                beta = txinputs.scalar(kind, 2) if general else 0
                it = [0]

                def gemm():
                    A, B, C = bufs[it[0] % sets]
                    it[0] += 1
                    rc = tx.tx_gemm_batched(kind, "N", "N", n, n, n, alpha, A, n, e, B, n, e, beta,
                                            C, n, e, batch)
                    assert rc == 0, tx.status_string(rc)

                def elementwise():  # same bytes: A, B (C) read, C written
                    A, B, C = bufs[it[0] % sets]
                    it[0] += 1
                    if general:
                        torch.addcmul(C, A, B, out=C)
                    else:
                        torch.mul(A, B, out=C)

                byts = model.bytes_moved(kind, n, n, n, batch, True, general)
                reps = 100
                tg = graph_time(gemm, reps)
                tr = graph_time(elementwise, reps)
                r = {"kind": kind, "n": n, "beta0": not general, "gemm_us": round(tg * 1e3, 3),
                     "torch_elementwise_us": round(tr * 1e3, 3),
                     "gemm_frac_hbm": round(byts / (tg / 1e3) / 1e9 / peak, 4),
                     "elementwise_frac_hbm": round(byts / (tr / 1e3) / 1e9 / peak, 4),
                     "gemm_over_elementwise": round(tr / tg, 4), "path": tx.last_path()[0],
                     "sets": sets}
                print(json.dumps(r), flush=True)
                if out:
                    out.write(json.dumps(r) + "\n")
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
