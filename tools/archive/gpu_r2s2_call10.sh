#!/bin/bash
# Round 2 (session 2), call 10: TC kernel v6 (complex as X [Br|Bi], 8 epilogue warps): parity, variants,
# A/B against the CUDA-core path over s 17-64 / c 9-32.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/s2c10_pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c10_pytest_tc.log
tail -3 gpurun_out/s2c10_pytest_tc.log
timeout 1200 bash tools/tc_variants.sh > gpurun_out/s2c10_variants.txt 2>&1
grep HBM gpurun_out/s2c10_variants.txt | grep "base\|noepi"
for t in 1 0; do
  TX_TC=$t timeout 1200 python tools/gate_run.py --kinds s --sizes 17-64 --ops NN,TT --out gpurun_out/s2c10_tcs${t}.jsonl 2>> gpurun_out/s2c10_gate.err
  TX_TC=$t timeout 900 python tools/gate_run.py --kinds c --sizes 9-32 --ops NN,CT,TC --out gpurun_out/s2c10_tcc${t}.jsonl 2>> gpurun_out/s2c10_gate.err
done
tail -4 gpurun_out/s2c10_gate.err
