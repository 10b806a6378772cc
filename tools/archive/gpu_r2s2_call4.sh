#!/bin/bash
# Round 2 (session 2), call 4: warp-specialised TC kernel parity + A/B + ncu; sustained DMMA A/B on
# the bench kernels (configs[4]); the default bench line with the DMMA table.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/s2c4_pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c4_pytest_tc.log
tail -3 gpurun_out/s2c4_pytest_tc.log
for t in 1 0 1; do
  TX_TC=$t timeout 1200 python tools/gate_run.py --kinds s --sizes 17-64 --ops NN,TT --out gpurun_out/s2c4_tcs${t}_$RANDOM.jsonl 2>> gpurun_out/s2c4_gate.err
  TX_TC=$t timeout 900 python tools/gate_run.py --kinds c --sizes 9-32 --ops NN,CT,TC --out gpurun_out/s2c4_tcc${t}_$RANDOM.jsonl 2>> gpurun_out/s2c4_gate.err
done
for d in 1 0 1 0; do
  TX_DMMA=$d timeout 900 python bench.py --steps 10 --warmup 3 --no-gate --no-sub --no-e2e --no-cpu > gpurun_out/s2c4_bench_dmma${d}_$RANDOM.json 2>> gpurun_out/s2c4_bench.err
done
timeout 1200 python bench.py --gate-out gpurun_out/s2c4_gate.jsonl > gpurun_out/s2c4_bench.json 2>> gpurun_out/s2c4_bench.err
TX_TC=1 PROF_REPS=1 timeout 600 ncu --set full --clock-control none -k regex:'tc_kernel' -o /tmp/ncu/tc -f \
  python tools/prof_list.py "s64NNgen c32NNgen c32NNb0 s40NNgen c13NNb0" 100000 > gpurun_out/s2c4_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/tc.ncu-rep > gpurun_out/s2c4_ncu_tc.json 2>> gpurun_out/s2c4_ncu.log
tail -8 gpurun_out/s2c4_gate.err; tail -3 gpurun_out/s2c4_bench.err; du -sh gpurun_out
