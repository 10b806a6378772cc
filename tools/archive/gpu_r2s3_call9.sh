#!/bin/bash
# Round 2 (session 3), call 9: compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the
# small cases of every kernel family incl. the bulk_ptr rings with a capped grid; s16/s10 at
# 10^5 pairs vs grid size (tail quantisation of the persistent grid).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh > gpurun_out/s3c9_sanitize.txt 2>&1
for f in gpurun_out/san_*.log; do mv $f gpurun_out/s3c9_$(basename $f); done
python - > gpurun_out/s3c9_grid.txt 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1304_7053_b200 as tx, txinputs
from paper_1304_7053_b200 import model
import json
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs']
for n in (10, 16):
    e = n * n; batch = 100000
    sets = [tuple(txinputs.values_torch('s', 100 + 3 * s + i, 0, e * batch, 'cuda') for i in range(3)) for s in range(2)]
    for cap in (0, 592, 576, 569, 560, 444, 296):
        tx.set_max_ctas(cap)
        it = [0]
        def call():
            A, B, C = sets[it[0] % 2]; it[0] += 1
            assert tx.tx_gemm_batched('s', 'N', 'N', n, n, n, 0.7, A, n, e, B, n, e, 0.3, C, n, e, batch) == 0
        for _ in range(20): call()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(200): call()
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 200
        byts = model.bytes_moved('s', n, n, n, batch, True, True)
        print(json.dumps({'n': n, 'max_ctas': cap, 'us': round(t * 1e3, 2), 'frac': round(byts / (t / 1e3) / 1e9 / peak, 4)}), flush=True)
    tx.set_max_ctas(0)
PY
cat gpurun_out/s3c9_sanitize.txt; cat gpurun_out/s3c9_grid.txt
