"""Per-(type, n) ncu table of the gate instances (measurement tool, not the product).

Reads the CSV that `ncu --csv --metrics ... --log-file F python tools/prof_list.py SPECS`
writes (one capture per launch, PROF_REPS=1) together with the spec list, and prints one
JSON line per instance: kernel, duration, DRAM bytes vs the algorithmic bytes, achieved DRAM
GB/s and its fraction of the measured peak, shared-memory wavefronts and bank conflicts per
pair, FMA / FP64 pipe and issue utilisation, SM clock.

  python tools/ncu_table.py ncu.csv "s1NNgen s1NNb0 ..." [BATCH] > table.jsonl
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1304_7053_b200 import model  # noqa: E402

path, specs = sys.argv[1], sys.argv[2].split()
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
by = {}
for r in rows:
    d = by.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"]})
    v = r["Metric Value"].replace(",", "")
    try:
        d[r["Metric Name"]] = float(v)
    except ValueError:
        d[r["Metric Name"]] = v
pat = re.compile(r"^([sdcz])(\d+)([NTC])([NTC])(b0|gen)$")
ids = sorted(by)
if len(ids) != len(specs):
    print(f"# {len(ids)} captures for {len(specs)} specs", file=sys.stderr)
for sp, i in zip(specs, ids):
    kind, n, ta, tb, b = pat.match(sp).groups()
    n = int(n)
    d = by[i]
    alg = model.bytes_moved(kind, n, n, n, batch, True, b == "gen")
    t_ns = d.get("gpu__time_duration.sum", 0.0)  # ns
    dram = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    out = {"spec": sp, "kernel": d["kernel"][:90], "us": round(t_ns / 1e3, 2),
           "alg_bytes": alg, "dram_bytes": dram,
           "dram_over_alg": round(dram / alg, 3) if alg else None,
           "alg_gbps": round(alg / t_ns, 1) if t_ns else None,
           "frac_of_measured_peak": round(alg / t_ns / peak, 4) if t_ns else None,
           "smem_ld_wavefronts_per_pair": round(d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 0) / batch, 1),
           "smem_ld_conflicts_per_pair": round(d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 0) / batch, 1),
           "fma_pipe_pct": d.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
           "fp64_pipe_pct": d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
           "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "sm_ghz": round(d.get("sm__cycles_elapsed.avg.per_second", 0) / 1e9, 3)}
    print(json.dumps(out))
