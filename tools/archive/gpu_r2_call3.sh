#!/bin/bash
# Round 2, call 3: the bench line (cfg5 + gate), direct A/B, ncu of gate misses (summaries only).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 900 python bench.py --gate-out gpurun_out/r2c3_gate.jsonl > gpurun_out/r2c3_bench.json 2> gpurun_out/r2c3_bench.err
echo "bench rc=$?" >> gpurun_out/r2c3_bench.err
for d in 1 0; do
  TX_DIRECT=$d timeout 300 python tools/sweep.py --kinds sdcz --sizes 1-2 --ops NN,NT,TN,TT,CN --graph \
    --out gpurun_out/r2c3_direct$d.jsonl > /dev/null 2>> gpurun_out/r2c3_sweep.err
done
PROF_REPS=1 timeout 900 ncu --set full -k regex:'bulk_kernel|direct_kernel' -o /tmp/ncu/miss -f \
  python tools/prof_list.py "s1NNb0 s1NNgen s2NNb0 d1NNb0 c1NNb0 z1NNb0 s3NTb0 c5NNb0 c7NTb0 c9CTb0 c13TCb0 c13NNb0 z14CTb0 z14NNb0 z16TTb0 z16CNb0 z11NNb0 z8NNb0" > gpurun_out/r2c3_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2c3_ncu.log
python tools/ncu_summary.py /tmp/ncu/miss.ncu-rep > gpurun_out/r2c3_ncu_summary.json 2>> gpurun_out/r2c3_ncu.log
ls -la /tmp/ncu >> gpurun_out/r2c3_ncu.log
du -sh gpurun_out
tail -2 gpurun_out/r2c3_bench.err; head -c 300 gpurun_out/r2c3_bench.json
