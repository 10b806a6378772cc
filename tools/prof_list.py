"""Run a list of strided square instances (for ncu), each twice at BATCH pairs.

  python tools/prof_list.py "c13NNb0 z14CTb0 s1NNb0 ..." [BATCH]

An instance spec is <kind><n><opA><opB><b0|gen>.  Under
  ncu --set full -k regex:'bulk_kernel|direct_kernel' --launch-skip 0 ...
every launch is captured; tools/ncu_summary.py then tabulates them.
"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1304_7053_b200 as tx  # noqa: E402
import txinputs  # noqa: E402

specs = sys.argv[1].split()
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
reps = int(os.environ.get("PROF_REPS", "2"))
pat = re.compile(r"^([sdcz])(\d+)([NTC])([NTC])(b0|gen)$")
for sp in specs:
    kind, n, ta, tb, b = pat.match(sp).groups()
    n = int(n)
    e = n * n
    A = txinputs.values_torch(kind, 1, 0, e * batch, "cuda")
    B = txinputs.values_torch(kind, 2, 0, e * batch, "cuda")
    C = txinputs.values_torch(kind, 3, 0, e * batch, "cuda")
    alpha = txinputs.scalar(kind, 11)
    beta = 0 if b == "b0" else txinputs.scalar(kind, 12)
    for _ in range(reps):
        rc = tx.tx_gemm_batched(kind, ta, tb, n, n, n, alpha, A, n, e, B, n, e, beta, C, n, e, batch)
        assert rc == 0, tx.status_string(rc)
    torch.cuda.synchronize()
    print(sp, tx.last_path(), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
