"""A/B of the pointer-array kernels (measurement tool, not the product).

For each shape and type: the pointer-array GEMM on seeded randomly permuted pointers
(BASELINE configs[3] recipe) at 10^6 pairs, CUDA-graph-timed over rotating buffer sets
>= 4 x L2, once per pipeline setting in --tunings ("S:KB" through tx_set_tuning, "0:0" =
the planner's own), plus the strided call of the same shape for reference.  Process-wide
choices (TX_PTR_BULK_MIN, TX_DMMA) are set in the environment and recorded as "tag".

  TX_PTR_BULK_MIN=1000000 python tools/ptr_ab.py --shapes 16x16x16 --out g16.jsonl
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
    ap.add_argument("--shapes", default="16x16x16")
    ap.add_argument("--kinds", default="sdcz")
    ap.add_argument("--ops", default="NN")
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--tunings", default="0:0")
    ap.add_argument("--strided", action="store_true")
    ap.add_argument("--tag", default="TX_PTR_BULK_MIN=%s TX_DMMA=%s" % (
        os.environ.get("TX_PTR_BULK_MIN", ""), os.environ.get("TX_DMMA", "")))
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = open(a.out, "a") if a.out else None
    for shp in a.shapes.split(","):
        m, n, k = (int(x) for x in shp.split("x"))
        for kind in a.kinds:
            es = model.ESIZE[kind]
            batch = a.batch
            sets = max(1, -(-4 * 126 * 2**20 // (es * (m * k + k * n + m * n) * batch)))
            bufs = []
            for s in range(sets):
                key = lambda nm: txinputs.stream_key(9, "ptrab", kind, m, n, k, s, nm)
                bufs.append(tuple(txinputs.values_torch(kind, key(nm), 0, e * batch, "cuda")
                                  for nm, e in (("A", m * k), ("B", k * n), ("C", m * n))))
            perm = torch.randperm(batch, generator=torch.Generator().manual_seed(3)).cuda()
            ptrs = [tuple(x.data_ptr() + perm * (e * es) for x, e in
                          zip(b, (m * k, k * n, m * n))) for b in bufs]
            alpha = txinputs.scalar(kind, 1)
            for ops in a.ops.split(","):
                ta, tb = ops[0], ops[1]
                lda = m if ta == "N" else k
                ldb = k if tb == "N" else n
                for general in (False, True):
                    beta = txinputs.scalar(kind, 2) if general else 0
                    byts = model.bytes_moved(kind, m, n, k, batch, True, general)
                    reps = int(max(4, min(100, 10.0 / (byts / (peak * 1e6)))))
                    variants = [("ptr", t) for t in a.tunings.split(",")]
                    if a.strided:
                        variants.append(("strided", "0:0"))
                    for layout, tun in variants:
                        S, KB = (int(x) for x in tun.split(":"))
                        tx.set_tuning(S, KB)
                        it = [0]

                        def call():
                            i = it[0] % sets
                            it[0] += 1
                            if layout == "ptr":
                                pa, pb, pc = ptrs[i]
                                rc = tx.tx_gemm_batched_ptr(kind, ta, tb, m, n, k, alpha, pa, lda,
                                                            pb, ldb, beta, pc, m, batch)
                            else:
                                A, B, C = bufs[i]
                                rc = tx.tx_gemm_batched(kind, ta, tb, m, n, k, alpha, A, lda,
                                                        m * k, B, ldb, k * n, beta, C, m, m * n,
                                                        batch)
                            assert rc == 0, tx.status_string(rc)

                        try:
                            t = graph_time(call, reps)
                        except AssertionError as ex:
                            print(json.dumps({"kind": kind, "shape": shp, "tuning": tun,
                                              "error": str(ex)}), flush=True)
                            continue
                        finally:
                            tx.set_tuning(0, 0)
                        r = {"kind": kind, "m": m, "n": n, "k": k, "ops": ops, "beta0": not general,
                             "layout": layout, "tuning": tun, "path": tx.last_path()[0], "jit": tx.binding.last_path_jit(),
                             "us": round(t * 1e3, 2),
                             "frac": round(byts / (t / 1e3) / 1e9 / peak, 4), "sets": sets,
                             "tag": a.tag}
                        print(json.dumps(r), flush=True)
                        if out:
                            out.write(json.dumps(r) + "\n")
            del bufs, ptrs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
