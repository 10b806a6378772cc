#!/bin/bash
# Round 2 (session 3), call 7: pointer-array gather preference (transposed A without DMMA, d/c
# general) -- pointer parity subset, A/B lines on the affected shapes, configs[3] sweep; then the
# default bench line and its launch list.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c7
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pointer or ptr" > gpurun_out/${P}_pytest_ptr.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest_ptr.log
timeout 600 python tools/ptr_ab.py --kinds zdc --shapes 16x3x16,8x16x4,16x16x16 --ops NN,TT,CN --tag rule --out gpurun_out/${P}_ptr_ab.jsonl > gpurun_out/${P}_ptr_ab.log 2>&1
timeout 1200 python tools/sweep.py --layout ptr --graph --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --ops NN,TT,TN,CC,CN --out gpurun_out/${P}_sweep_ptr.jsonl > gpurun_out/${P}_sweep_ptr.log 2>&1
echo "sweep rc=$?" >> gpurun_out/${P}_sweep_ptr.log
timeout 1200 python bench.py --gate-out gpurun_out/${P}_gate.jsonl > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
echo "bench rc=$?" >> gpurun_out/${P}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bulk_kernel|gather_kernel|scale_kernel|direct_kernel' -c 40 --csv \
  --log-file gpurun_out/${P}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/${P}_launch_bench.log 2>&1
tail -3 gpurun_out/${P}_pytest_ptr.log; tail -1 gpurun_out/${P}_sweep_ptr.log; tail -1 gpurun_out/${P}_bench.err; head -c 300 gpurun_out/${P}_bench.json; du -sh gpurun_out
