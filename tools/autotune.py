"""Autotune the pipeline depth S and stage size (KB) of every size-specialised bulk
instance on the GPU (tx_set_tuning), at 10^6 pairs per call, all op pairs, beta = 0 and
general.  Writes one JSON line per (instance, S, KB) measurement.

  python tools/autotune.py --out gpurun_out/autotune.jsonl [--kinds sdcz] [--sizes 1-16]"""
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

L2 = 126 * 1024 * 1024
CONFIGS = [(s, kb) for s in (2, 3, 4) for kb in (8, 16, 32)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="sdcz")
    ap.add_argument("--sizes", default="1-16")
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    lo, hi = (int(x) for x in a.sizes.split("-"))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = open(a.out, "a")
    batch = a.batch
    for kind in a.kinds:
        ops = ["N", "T", "C"] if kind in "cz" else ["N", "T"]
        for n in range(lo, hi + 1):
            es = model.ESIZE[kind]
            per_set = es * 3 * n * n * batch
            R = max(1, min(6, -(-4 * L2 // per_set)))
            sets = []
            for r in range(R):
                key = lambda nm: txinputs.stream_key(9, "tune", kind, n, r, nm)
                sets.append([txinputs.values_torch(kind, key(nm), 0, n * n * batch, "cuda")
                             for nm in "ABC"])
            alpha, beta = txinputs.scalar(kind, 21), txinputs.scalar(kind, 22)
            for ta in ops:
                for tb in ops:
                    for b0 in (True, False):
                        bb = 0 if b0 else beta

                        def call(i):
                            A, B, C = sets[i % R]
                            rc = tx.tx_gemm_batched(kind, ta, tb, n, n, n, alpha, A, n, n * n, B,
                                                    n, n * n, bb, C, n, n * n, batch)
                            assert rc == 0
                        byts = model.bytes_moved(kind, n, n, n, batch, True, not b0)
                        for S, kb in CONFIGS:
                            tx.set_tuning(S, kb)
                            for i in range(R + 1):
                                call(i)
                            e0 = torch.cuda.Event(enable_timing=True)
                            e1 = torch.cuda.Event(enable_timing=True)
                            e0.record()
                            for i in range(a.reps):
                                call(i)
                            e1.record()
                            torch.cuda.synchronize()
                            ms = e0.elapsed_time(e1) / a.reps
                            gbps = byts / (ms / 1e3) / 1e9
                            out.write(json.dumps({"kind": kind, "n": n, "ops": ta + tb, "beta0": b0,
                                                  "S": S, "KB": kb, "frac": round(gbps / peak, 4),
                                                  "us": round(ms * 1e3, 2)}) + "\n")
                        tx.set_tuning(0, 0)
            out.flush()
            del sets
            torch.cuda.empty_cache()
            print(kind, n, "done", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
