"""Set the TRA column of csrc/tx_map_table.inc where the transpose-at-staging build
measured faster (> 3 %) than the current table.
  python tools/apply_tra.py current_sweep.jsonl tra_sweep.jsonl"""
import json
import re
import sys

TABLE = "paper_1304_7053_b200/csrc/tx_map_table.inc"
KIND = {"s": "float", "d": "double", "c": "float2", "z": "double2"}
OPC = {"N": 0, "T": 1, "C": 2}


def load(path):
    d = {}
    for line in open(path):
        r = json.loads(line)
        d[(KIND[r["kind"]], r["n"], OPC[r["ops"][0]], OPC[r["ops"][1]], 1 if r["beta0"] else 0)] = r["frac_measured"]
    return d


cur, tra = load(sys.argv[1]), load(sys.argv[2])
out, flips = [], []
for line in open(TABLE).read().splitlines():
    m = re.match(r"TX_MAP\(([^)]*)\)(.*)", line)
    if not m:
        out.append(line)
        continue
    f = [x.strip() for x in m.group(1).split(",")]
    key = (f[0], int(f[1]), int(f[2]), int(f[3]), int(f[4]))
    if key in tra and key in cur and tra[key] > cur[key] * 1.03 and key[2] != 0:
        f[16] = "1"
        flips.append((key, cur[key], tra[key]))
        out.append(f"TX_MAP({', '.join(f)}) // TRA measured {tra[key]:.3f} (was {cur[key]:.3f})")
    else:
        out.append(line)
open(TABLE, "w").write("\n".join(out) + "\n")
print("TRA on for", len(flips), "instances")
for k, a, b in sorted(flips, key=lambda t: t[1])[:30]:
    print(k, round(a, 3), "->", round(b, 3))
