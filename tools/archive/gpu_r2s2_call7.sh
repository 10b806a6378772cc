#!/bin/bash
# Round 2 (session 2), call 7: TC kernel v4 (separate A/B and C rings) variants, traces, probe.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py > gpurun_out/s2c7_tcprobe.json 2> gpurun_out/s2c7_tcprobe.err
timeout 1200 bash tools/tc_variants.sh > gpurun_out/s2c7_variants.txt 2>&1
for c in "c 32 32 32 gen" "s 64 64 64 gen" "c 24 24 24 b0"; do
  echo "== $c" >> gpurun_out/s2c7_trace.txt
  timeout 300 python tools/tc_trace.py $c >> gpurun_out/s2c7_trace.txt 2>&1
done
cat gpurun_out/s2c7_variants.txt; grep "steady\|HBM" gpurun_out/s2c7_trace.txt
