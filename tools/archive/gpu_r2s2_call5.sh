#!/bin/bash
# Round 2 (session 2), call 5: timeline of the TC kernel (tools/tc_trace.py), s sizes 17-64 gate
# diagnosis (per-size errors recorded).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for c in "c 32 32 32 gen" "s 64 64 64 gen" "c 24 24 24 b0" "s 40 40 40 gen"; do
  echo "== $c" >> gpurun_out/s2c5_trace.txt
  timeout 300 python tools/tc_trace.py $c >> gpurun_out/s2c5_trace.txt 2>&1
done
for t in 1 0; do
  TX_TC=$t timeout 900 python tools/gate_run.py --kinds s --sizes 17-64 --ops NN --out gpurun_out/s2c5_tcs${t}.jsonl 2>> gpurun_out/s2c5_gate.err
done
grep -v "^\s*[0-9]* *-1" gpurun_out/s2c5_trace.txt | head -120; grep -i "rc=\|instances" gpurun_out/s2c5_gate.err | head -20
