"""Write the autotuned (S, KB) of every instance into csrc/tx_map_table.inc.

  python tools/apply_autotune.py gpurun_out/autotune.jsonl [more.jsonl ...]
A config must beat the current table entry's own config by > 1 % to replace it."""
import json
import re
import statistics
import sys
from collections import defaultdict

TABLE = "paper_1304_7053_b200/csrc/tx_map_table.inc"
KIND = {"s": "float", "d": "double", "c": "float2", "z": "double2"}
OPC = {"N": 0, "T": 1, "C": 2}

res = defaultdict(dict)
for path in sys.argv[1:]:
    for line in open(path):
        r = json.loads(line)
        key = (KIND[r["kind"]], r["n"], OPC[r["ops"][0]], OPC[r["ops"][1]], 1 if r["beta0"] else 0)
        res[key].setdefault((r["S"], r["KB"]), []).append(r["frac"])

lines = open(TABLE).read().splitlines()
out, gains = [], []
for line in lines:
    m = re.match(r"TX_MAP\(([^)]*)\)(.*)", line)
    if not m:
        out.append(line)
        continue
    f = [x.strip() for x in m.group(1).split(",")]
    key = (f[0], int(f[1]), int(f[2]), int(f[3]), int(f[4]))
    if key not in res:
        out.append(line)
        continue
    meas = {c: max(v) for c, v in res[key].items()}
    cur = (int(f[14]) or 4, int(f[15]) or 16)
    cur_v = meas.get(cur, max(meas.values()))
    best_c, best_v = max(meas.items(), key=lambda kv: kv[1])
    if best_v <= cur_v * 1.01:
        best_c, best_v = cur, cur_v
    f[14], f[15] = str(best_c[0]), str(best_c[1])
    gains.append((best_v, cur_v, key))
    out.append(f"TX_MAP({', '.join(f)}) // autotuned {best_v:.3f} (S={best_c[0]}, {best_c[1]} KB)")
open(TABLE, "w").write("\n".join(out) + "\n")
vals = [g[0] for g in gains]
print("instances", len(gains), "median", statistics.median(vals), "min", min(vals),
      "below .70", sum(v < 0.70 for v in vals), "below .855", sum(v < 0.855 for v in vals))
print("improved >5%:", sum(1 for b, c, k in gains if b > c * 1.05))
for b, c, k in sorted(gains)[:40]:
    if k[1] > 2:
        print(k, round(c, 3), "->", round(b, 3))
