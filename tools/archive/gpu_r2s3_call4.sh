#!/bin/bash
# Round 2 (session 3), call 4: pointer-array dispatch after the A/B (bulk_ptr: 2 x 16 KB stages,
# decoupled ring for d/c/z general, no DMMA for skinny pointer shapes): pointer parity tests,
# configs[3] sweep (same protocol as round 1's r01_sweep_ptr_v8), A/B lines, default bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c4
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pointer or ptr" > gpurun_out/${P}_pytest_ptr.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest_ptr.log
timeout 900 python tools/ptr_ab.py --shapes 16x16x16,16x3x16,8x16x4,1x16x16,4x6x16,16x16x1,5x7x3 --ops NN,TT --strided --tag s3c4 --out gpurun_out/${P}_ptr_ab.jsonl > gpurun_out/${P}_ptr_ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/${P}_ptr_ab.log
timeout 1200 python tools/sweep.py --layout ptr --graph --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --ops NN,TT,TN,CC,CN --out gpurun_out/${P}_sweep_ptr.jsonl > gpurun_out/${P}_sweep_ptr.log 2>&1
echo "sweep rc=$?" >> gpurun_out/${P}_sweep_ptr.log
timeout 1200 python bench.py --gate-out gpurun_out/${P}_gate.jsonl > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
echo "bench rc=$?" >> gpurun_out/${P}_bench.err
tail -3 gpurun_out/${P}_pytest_ptr.log; tail -1 gpurun_out/${P}_ptr_ab.log; tail -1 gpurun_out/${P}_sweep_ptr.log; tail -1 gpurun_out/${P}_bench.err; head -c 300 gpurun_out/${P}_bench.json; du -sh gpurun_out
