#!/bin/bash
# Round 2, call 4: DMMA semantics/throughput probe; pointer-pattern roof; ncu (clocks unlocked) of the bench kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/dmma_probe.py > gpurun_out/r2c4_dmma.json 2> gpurun_out/r2c4_dmma.err
timeout 900 python tools/ptr_roof.py --out gpurun_out/r2c4_ptr_roof.jsonl > /dev/null 2> gpurun_out/r2c4_ptr_roof.err
PROF_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'bulk_kernel' -o /tmp/ncu/bench -f \
  python tools/prof_list.py "z16NNgen d16NNgen s16NNgen s10NNgen" > gpurun_out/r2c4_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/bench.ncu-rep > gpurun_out/r2c4_ncu_bench.json 2>> gpurun_out/r2c4_ncu.log
cp /tmp/ncu/bench.ncu-rep gpurun_out/r2c4_bench_kernels.ncu-rep
PROF_REPS=1 timeout 900 ncu --set full --clock-control none -k regex:'bulk_kernel' -o /tmp/ncu/miss -f \
  python tools/prof_list.py "c13CCb0 c13TCb0 c16TNb0 z16TNb0 z14NNb0 z13NNb0 d15NTb0 d13NNb0 z8NNb0 s13NNb0" > gpurun_out/r2c4_ncu2.log 2>&1
python tools/ncu_summary.py /tmp/ncu/miss.ncu-rep > gpurun_out/r2c4_ncu_miss.json 2>> gpurun_out/r2c4_ncu2.log
du -sh gpurun_out; cat gpurun_out/r2c4_dmma.json; tail -3 gpurun_out/r2c4_ptr_roof.err
