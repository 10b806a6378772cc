"""Run bench.py's gate sweep on a subset (A/B measurements of kernel variants).

  TX_DMMA=1 python tools/gate_run.py --kinds dz --sizes 1-16 --out on.jsonl
  TX_TC=0   python tools/gate_run.py --kinds sc --sizes 17,24,32 --ops NN,TT --out off.jsonl

Same protocol as the bench's "gate" record: CUDA-graph-replayed back-to-back calls over
rotating buffer sets >= 4 x L2, fraction of the measured HBM peak (sizes > 16 use fewer
pairs so one operand fits the 4 GB pool).  One JSON line per instance (+ "tag")."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def sizes_of(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="sdcz")
    ap.add_argument("--sizes", default="1-16")
    ap.add_argument("--ops", default="", help="comma list, e.g. NN,TT (default: all)")
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--tag", default=os.environ.get("TX_DMMA", "") + "/" + os.environ.get("TX_TC", ""))
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    peak, _ = bench.peaks()
    res, wall = [], 0.0
    for kind in a.kinds:
        for n in sizes_of(a.sizes):
            try:
                r, w = bench.gate_sweep("cuda:0", peak, batch=a.batch, kinds=kind, sizes=[n],
                                        ops_filter=set(a.ops.split(",")) if a.ops else None)
                res += r
                wall += w
            except AssertionError as e:  # a failing call: record it, go on
                res.append({"kind": kind, "n": n, "error": str(e)})
                print(f"{kind}{n}: {e}", file=sys.stderr)
    with open(a.out, "w") as f:
        for r in res:
            r["tag"] = a.tag
            f.write(json.dumps(r) + "\n")
    print(f"{len(res)} instances in {wall:.1f} s -> {a.out}", file=sys.stderr)


if __name__ == "__main__":
    main()
