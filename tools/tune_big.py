"""Pipeline-setting sweep of the runtime-specialised strided instances beyond 16
(measurement tool, not the product): for each type and square size, the strided call under
each (S stages, stage KB) of --tunings (tx_set_tuning; "0:0" = the planner's own), CUDA-graph-
timed over rotating buffer sets >= 4 x L2 (the gate protocol).  One JSON line per case.

  python tools/tune_big.py --kinds s --sizes 24,32,40 --out tune.jsonl
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

sys.path.insert(0, os.path.join(ROOT, "tools"))
from ptr_ab import graph_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="sc")
    ap.add_argument("--sizes", default="24,32")
    ap.add_argument("--ops", default="NN")
    ap.add_argument("--tunings", default="0:0,2:16,2:32,3:32,2:64,3:64,4:32")
    ap.add_argument("--bytes", type=float, default=1.2e9, help="operand bytes per set (A+B+C)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = open(a.out, "a") if a.out else None
    for kind in a.kinds:
        for n in (int(x) for x in a.sizes.split(",")):
            es = model.ESIZE[kind]
            e = n * n
            batch = int(a.bytes // (3 * e * es))
            sets = max(1, -(-4 * 126 * 2**20 // (3 * e * es * batch)))
            bufs = [tuple(txinputs.values_torch(kind, txinputs.stream_key(11, "tune", kind, n, s, nm),
                                                0, e * batch, "cuda") for nm in "ABC")
                    for s in range(sets)]
            alpha = txinputs.scalar(kind, 1)
            for ops in a.ops.split(","):
                for general in (False, True):
                    beta = txinputs.scalar(kind, 2) if general else 0
                    byts = model.bytes_moved(kind, n, n, n, batch, True, general)
                    for tun in a.tunings.split(","):
                        S, KB = (int(x) for x in tun.split(":"))
                        tx.set_tuning(S, KB)
                        it = [0]

                        def call():
                            A, B, C = bufs[it[0] % sets]
                            it[0] += 1
                            rc = tx.tx_gemm_batched(kind, ops[0], ops[1], n, n, n, alpha, A, n, e,
                                                    B, n, e, beta, C, n, e, batch)
                            assert rc == 0, tx.status_string(rc)

                        try:
                            t = graph_time(call, 10)
                        finally:
                            tx.set_tuning(0, 0)
                        r = {"kind": kind, "n": n, "ops": ops, "beta0": not general, "tuning": tun,
                             "batch": batch, "path": tx.last_path()[0], "us": round(t * 1e3, 2),
                             "frac": round(byts / (t / 1e3) / 1e9 / peak, 4)}
                        print(json.dumps(r), flush=True)
                        if out:
                            out.write(json.dumps(r) + "\n")
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
