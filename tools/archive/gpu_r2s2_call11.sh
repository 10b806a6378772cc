#!/bin/bash
# Round 2 (session 2), call 11: TC kernel v7 (epilogue without per-element index math, plan prefers
# A/B bytes in flight): parity, variants, A/B.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/s2c11_pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c11_pytest_tc.log
tail -3 gpurun_out/s2c11_pytest_tc.log
timeout 1200 bash tools/tc_variants.sh > gpurun_out/s2c11_variants.txt 2>&1
grep HBM gpurun_out/s2c11_variants.txt
TX_TC=1 timeout 1200 python tools/gate_run.py --kinds s --sizes 17-64 --ops NN,TT --out gpurun_out/s2c11_tcs1.jsonl 2>> gpurun_out/s2c11_gate.err
TX_TC=1 timeout 900 python tools/gate_run.py --kinds c --sizes 9-32 --ops NN,CT,TC --out gpurun_out/s2c11_tcc1.jsonl 2>> gpurun_out/s2c11_gate.err
tail -4 gpurun_out/s2c11_gate.err
