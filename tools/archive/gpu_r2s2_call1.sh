#!/bin/bash
# Round 2 (session 2), call 1: full GPU suite + smoke, the default bench line (cfg5 + gate),
# the bench launch list, and an ncu --set full capture of the bench kernels (d16/z16 general).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2c1_nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=30 > gpurun_out/s2c1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2c1_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s2c1_smoke.log
timeout 1200 python bench.py --gate-out gpurun_out/s2c1_gate.jsonl > gpurun_out/s2c1_bench.json 2> gpurun_out/s2c1_bench.err
echo "bench rc=$?" >> gpurun_out/s2c1_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bulk_kernel|gather_kernel|scale_kernel|direct_kernel' -c 40 --csv \
  --log-file gpurun_out/s2c1_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/s2c1_launch_bench.log 2>&1
echo "ncu-list rc=$?" >> gpurun_out/s2c1_launch_bench.log
PROF_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bulk_kernel' -o /tmp/ncu/bench -f \
  python tools/prof_list.py "z16NNgen d16NNgen s16NNgen s10NNgen" > gpurun_out/s2c1_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s2c1_ncu.log
python tools/ncu_summary.py /tmp/ncu/bench.ncu-rep > gpurun_out/s2c1_ncu_bench.json 2>> gpurun_out/s2c1_ncu.log
cp /tmp/ncu/bench.ncu-rep gpurun_out/s2c1_bench_kernels.ncu-rep
tail -4 gpurun_out/s2c1_pytest.log; tail -3 gpurun_out/s2c1_smoke.log; tail -2 gpurun_out/s2c1_bench.err; head -c 400 gpurun_out/s2c1_bench.json; du -sh gpurun_out
