"""Set the ON column of csrc/tx_asw_table.inc from an A/B sweep: the ASW instance is
enabled where the build with it measured > 1.03 x the build without it (same box,
same call; tools/gpu_call_r1d.sh).  usage: apply_asw.py ASW.jsonl NOASW.jsonl"""
import json
import re
import sys

TN = {"double": "d", "float2": "c", "double2": "z"}
OPS = "NTC"


def load(f):
    return {(r["kind"], r["n"], r["ops"], r["beta0"]): r["frac_measured"] for r in map(json.loads, open(f))}


def main():
    a, b = load(sys.argv[1]), load(sys.argv[2])
    path = "paper_1304_7053_b200/csrc/tx_asw_table.inc"
    out = []
    for line in open(path):
        m = re.match(r"TX_ASWMAP\((\w+), (\d+), (\d), (\d), (\d), (.*), (\d)\)(.*)", line)
        if not m:
            out.append(line)
            continue
        t, n, oa, ob, b0 = m.group(1), int(m.group(2)), int(m.group(3)), int(m.group(4)), int(m.group(5))
        key = (TN[t], n, OPS[oa] + OPS[ob], b0 == 1)
        on = int(key in a and key in b and a[key] > 1.03 * b[key])
        note = f" // measured {a.get(key, 0):.3f} vs {b.get(key, 0):.3f} without" if key in a else ""
        out.append(f"TX_ASWMAP({t}, {n}, {oa}, {ob}, {b0}, {m.group(6)}, {on}){note}\n")
    open(path, "w").writelines(out)


if __name__ == "__main__":
    main()
