"""Set the ON column of csrc/tx_tra_table.inc (TRA instances' own searched mappings) where
the build with every entry on measured > 1.03 x the shipped mapping, averaged over two
interleaved runs each (cur, tra, cur, tra on one box; tools/gpu_call_r1z.sh).
usage: merge_tra.py CUR1 TRA1 CUR2 TRA2"""
import json
import re
import sys

TN = {"float": "s", "double": "d", "float2": "c", "double2": "z"}
OPS = "NTC"


def load(f):
    return {(r["kind"], r["n"], r["ops"], r["beta0"]): r["frac_measured"] for r in map(json.loads, open(f))}


def main():
    c1, t1, c2, t2 = (load(f) for f in sys.argv[1:5])
    path = "paper_1304_7053_b200/csrc/tx_tra_table.inc"
    out, n = [], 0
    for line in open(path):
        m = re.match(r"(TX_TRAMAP\((\w+), (\d+), (\d), (\d), (\d), .*), (\d)\) //(.*)", line)
        if not m:
            out.append(line)
            continue
        t, nn, oa, ob, b0 = m.group(2), int(m.group(3)), int(m.group(4)), int(m.group(5)), m.group(6)
        key = (TN[t], nn, OPS[oa] + OPS[ob], b0 == "1")
        on = 0
        note = m.group(8).split(" | measured")[0]
        if key in c1 and key in t1:
            cur, new = (c1[key] + c2[key]) / 2, (t1[key] + t2[key]) / 2
            on = int(new > 1.03 * cur)
            n += on
            note += f" | measured {new:.3f} vs {cur:.3f}"
        out.append(f"{m.group(1)}, {on}) //{note}\n")
    open(path, "w").writelines(out)
    print("enabled", n)


if __name__ == "__main__":
    main()
