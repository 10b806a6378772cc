"""Write csrc/tx_mma_table.inc: the FP64 tensor-core (DMMA) square instances' own
pipeline settings and whether each one is used.

  python tools/apply_mma.py --autotune at.jsonl [...] [--ab-on on1.jsonl on2.jsonl
                             --ab-off off1.jsonl off2.jsonl] [--margin 1.02]

--autotune: tools/autotune.py lines measured with TX_DMMA=1 (every (S, KB) per
instance); the best config is kept (ties within 1 % go to the fewer-stage one).
--ab-on / --ab-off: tools/sweep.py lines of the same box with TX_DMMA=1 / TX_DMMA=0
(interleaved runs, averaged); ON = 1 where the tensor-core instance measured more
than `margin` x the FMA instance.  Without A/B files every ON is 0.
"""
import argparse
import json
import statistics
from collections import defaultdict

TABLE = "paper_1304_7053_b200/csrc/tx_mma_table.inc"
KIND = {"d": "double", "z": "double2"}
OPC = {"N": 0, "T": 1, "C": 2}


def key_of(r):
    return (r["kind"], r["n"], r["ops"], r["beta0"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--autotune", nargs="*", default=[],
                    help="autotune lines; without them S, KB are kept from the current table")
    ap.add_argument("--ab-on", nargs="*", default=[])
    ap.add_argument("--ab-off", nargs="*", default=[])
    ap.add_argument("--margin", type=float, default=1.02)
    a = ap.parse_args()
    tune = defaultdict(lambda: defaultdict(list))
    if not a.autotune:  # keep the table's (S, KB); only the ON column is re-decided
        import re
        rx = re.compile(r"TX_MMAMAP\((\w+), (\d+), (\d), (\d), (\d), (\d+), (\d+), \d\)")
        name = {v: k for k, v in KIND.items()}
        opn = {v: k for k, v in OPC.items()}
        for line in open(TABLE):
            mt = rx.search(line)
            if mt:
                t, n, oa, ob, b0, S, KB = mt.groups()
                key = (name[t], int(n), opn[int(oa)] + opn[int(ob)], b0 == "1")
                tune[key][(int(S), int(KB))].append(1.0)
    for path in a.autotune:
        for line in open(path):
            r = json.loads(line)
            if r["kind"] in KIND:
                tune[key_of(r)][(r["S"], r["KB"])].append(r["frac"])

    def avg(paths):
        acc = defaultdict(list)
        for path in paths:
            for line in open(path):
                r = json.loads(line)
                acc[key_of(r)].append(r.get("frac_measured", r.get("frac")))
        return {k: statistics.mean(v) for k, v in acc.items()}

    on, off = avg(a.ab_on), avg(a.ab_off)
    lines = ["// TX_MMAMAP(T, n, OPA, OPB, B0, S, KB, ON): FP64 tensor-core square instances "
             "(tools/apply_mma.py)",
             "// S, KB: best of tools/autotune.py with TX_DMMA=1; ON: interleaved A/B "
             f"(TX_DMMA=1 vs 0) > {a.margin} x"]
    n_on = 0
    for k in sorted(tune):
        kind, n, ops, b0 = k
        meas = {c: max(v) for c, v in tune[k].items()}
        best = max(meas.values())
        cfg = min((c for c, v in meas.items() if v >= 0.99 * best), key=lambda c: (c[0], c[1]))
        flag = 1 if (k in on and k in off and on[k] > a.margin * off[k]) else 0
        n_on += flag
        note = (f"mma {on[k]:.3f} vs fma {off[k]:.3f}" if k in on and k in off
                else f"autotuned {meas[cfg]:.3f}")
        lines.append(f"TX_MMAMAP({KIND[kind]}, {n}, {OPC[ops[0]]}, {OPC[ops[1]]}, {1 if b0 else 0}, "
                     f"{cfg[0]}, {cfg[1]}, {flag}) // {note}")
    open(TABLE, "w").write("\n".join(lines) + "\n")
    print(f"{len(tune)} instances, {n_on} on")


if __name__ == "__main__":
    main()
