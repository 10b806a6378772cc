#!/bin/bash
# Round 2 (session 3), call 10: resident CTAs per SM of the persistent grids (TX_CTAS_PER_SM=2/3 vs
# the occupancy maximum): interleaved gate sweeps and bench lines; pipeline sweep of the
# runtime-specialised sizes beyond 16.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c10
export TX_JIT_CACHE=/tmp/txjit_$$
for r in 1 2; do
  for c in 0 2 3; do
    TX_CTAS_PER_SM=$c timeout 600 python tools/gate_run.py --tag cps$c --out gpurun_out/${P}_gate_cps${c}_$r.jsonl >> gpurun_out/${P}_gate.log 2>&1
  done
done
for r in 1 2; do
  for c in 0 2; do
    TX_CTAS_PER_SM=$c timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/${P}_bench_cps${c}_$r.json 2>> gpurun_out/${P}_bench.err
  done
done
timeout 900 python tools/tune_big.py --kinds s --sizes 24,32,40,48,56 --out gpurun_out/${P}_tune_big.jsonl > gpurun_out/${P}_tune_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds c --sizes 17,20,24,28 --out gpurun_out/${P}_tune_big.jsonl >> gpurun_out/${P}_tune_big.log 2>&1
tail -3 gpurun_out/${P}_gate.log; tail -2 gpurun_out/${P}_bench.err; tail -2 gpurun_out/${P}_tune_big.log; du -sh gpurun_out
