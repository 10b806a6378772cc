"""Merge the power-capped re-search (csrc/tx_map_table_pc.inc, tools/mapsearch.cpp --pc)
into csrc/tx_map_table.inc where it measured > 1.03 x the current entry, averaged over two
interleaved runs each (cur, pc, cur, pc on one box; tools/gpu_call_r1o.sh).  An op(A) = N
entry is not replaced when a TRA instance (op(A) = T/C, same op(B) and epilogue, no ASW)
borrows its mapping (tx_dispatch.cuh TraMap): the c14 NC beta = 0 entry once did, and its
CC / TC twins fell from 0.85 to 0.52.  A TRA entry itself is not replaced either (its measured
rate came from the candidate N entry's mapping, which may not be merged).
usage: merge_pc.py CUR1 PC1 CUR2 PC2"""
import json
import re
import sys

TN = {"float": "s", "double": "d", "float2": "c", "double2": "z"}
OPS = "NTC"


def load(f):
    return {(r["kind"], r["n"], r["ops"], r["beta0"]): r["frac_measured"] for r in map(json.loads, open(f))}


def main():
    c1, p1, c2, p2 = (load(f) for f in sys.argv[1:5])
    pat = re.compile(r"TX_MAP\((\w+), (\d+), (\d), (\d), (\d), ")
    pc_lines = {pat.match(l).groups(): l for l in open("tools/archive/tables/tx_map_table_pc.inc")
                if pat.match(l)}
    tra = set()  # (T, n, opb, b0) whose op(A) = N mapping a TRA instance borrows
    asw = {m.groups()[:5] for m in (re.match(r"TX_ASWMAP\((\w+), (\d+), (\d), (\d), (\d), .*, 1\)", l)
                                    for l in open("paper_1304_7053_b200/csrc/tx_asw_table.inc")) if m}
    for l in open("paper_1304_7053_b200/csrc/tx_map_table.inc"):
        m = re.match(r"TX_MAP\((\w+), (\d+), (\d), (\d), (\d), .*, 1\)", l)
        if m and m.group(3) != "0" and m.groups()[:5] not in asw:
            tra.add((m.group(1), m.group(2), m.group(4), m.group(5)))
    path = "paper_1304_7053_b200/csrc/tx_map_table.inc"
    out, n = [], 0
    for line in open(path):
        m = pat.match(line)
        if m:
            t, nn, oa, ob, b0 = m.groups()
            key = (TN[t], int(nn), OPS[int(oa)] + OPS[int(ob)], b0 == "1")
            own_tra = line.split(" //")[0].rstrip().endswith(", 1)") and m.groups()[:5] not in asw
            if key in c1 and key in p1 and not own_tra and not (oa == "0" and (t, nn, ob, b0) in tra):
                cur = (c1[key] + c2[key]) / 2
                new = (p1[key] + p2[key]) / 2
                if new > 1.03 * cur:
                    body = pc_lines[m.groups()].split(" //")[0]
                    line = f"{body} // pc search, measured {new:.3f} vs {cur:.3f}\n"
                    n += 1
        out.append(line)
    open(path, "w").writelines(out)
    print("merged", n)


if __name__ == "__main__":
    main()
