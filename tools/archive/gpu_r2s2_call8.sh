#!/bin/bash
# Round 2 (session 2), call 8: TC kernel with the cheaper split (tf32_hi, lo unrounded): variant timings,
# and an ncu source-level capture (per-SASS stall samples) of the c24 b0 and c32 gen launches.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 1200 bash tools/tc_variants.sh > gpurun_out/s2c8_variants.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -I include -I paper_1304_7053_b200/csrc -shared -Xcompiler -fPIC -o /tmp/tcli.so tools/tc_trace.cu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_kernel -c 1 -o /tmp/ncu/c24 -f \
  python tools/tc_trace.py c 24 24 24 b0 100000 --so /tmp/tcli.so --quiet > gpurun_out/s2c8_ncu.log 2>&1
ncu -i /tmp/ncu/c24.ncu-rep --page source --csv --print-source sass > gpurun_out/s2c8_src_c24.csv 2>> gpurun_out/s2c8_ncu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_kernel -c 1 -o /tmp/ncu/c32 -f \
  python tools/tc_trace.py c 32 32 32 gen 100000 --so /tmp/tcli.so --quiet >> gpurun_out/s2c8_ncu.log 2>&1
ncu -i /tmp/ncu/c32.ncu-rep --page source --csv --print-source sass > gpurun_out/s2c8_src_c32.csv 2>> gpurun_out/s2c8_ncu.log
python tools/ncu_summary.py /tmp/ncu/c24.ncu-rep > gpurun_out/s2c8_ncu_c24.json 2>> gpurun_out/s2c8_ncu.log
ls -la gpurun_out/; grep -v Remark gpurun_out/s2c8_variants.txt | grep HBM
