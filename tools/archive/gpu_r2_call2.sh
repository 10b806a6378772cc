#!/bin/bash
# Round 2, call 2: direct-kernel parity, the new bench line (cfg5 + gate), direct A/B, ncu of gate misses.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ring.py -m gpu -q -x -p no:cacheprovider \
  -k "direct or square_sweep or batch_edges or integer or ring_square" > gpurun_out/r2c2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c2_pytest.log
timeout 900 python bench.py --gate-out gpurun_out/r2c2_gate.jsonl > gpurun_out/r2c2_bench.json 2> gpurun_out/r2c2_bench.err
echo "bench rc=$?" >> gpurun_out/r2c2_bench.err
for d in 1 0; do
  TX_DIRECT=$d timeout 300 python tools/sweep.py --kinds sdcz --sizes 1-2 --ops NN,NT,TN,TT,CN --graph \
    --out gpurun_out/r2c2_direct$d.jsonl > /dev/null 2>> gpurun_out/r2c2_sweep.err
done
timeout 600 ncu --set full -k regex:'bulk_kernel|direct_kernel' -o gpurun_out/r2c2_miss -f \
  python tools/prof_list.py "s1NNb0 s1NNgen s2NNb0 d1NNb0 c1NNb0 z1NNb0 s3NTb0 c5NNb0 c7NTb0 c9CTb0 c13TCb0 c13NNb0 z14CTb0 z14NNb0 z16TTb0 z16CNb0 z11NNb0 z8NNb0" > gpurun_out/r2c2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2c2_ncu.log
tail -3 gpurun_out/r2c2_pytest.log; tail -2 gpurun_out/r2c2_bench.err; head -c 600 gpurun_out/r2c2_bench.json
