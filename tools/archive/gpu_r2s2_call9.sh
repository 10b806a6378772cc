#!/bin/bash
# Round 2 (session 2), call 9: TC kernel v5 (division-free rings, 8 epilogue warps): variants + trace.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 bash tools/tc_variants.sh > gpurun_out/s2c9_variants.txt 2>&1
for c in "c 32 32 32 gen" "s 64 64 64 gen" "c 24 24 24 b0"; do
  echo "== $c" >> gpurun_out/s2c9_trace.txt
  timeout 300 python tools/tc_trace.py $c >> gpurun_out/s2c9_trace.txt 2>&1
done
grep HBM gpurun_out/s2c9_variants.txt; grep "steady\|HBM" gpurun_out/s2c9_trace.txt
