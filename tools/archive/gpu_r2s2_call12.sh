#!/bin/bash
# Round 2 (session 2), call 12: checkpoint -- full GPU suite + smoke, the default bench line (configs[4] +
# gate + cfg2), its launch list, ncu --set full of the bench kernels (d16/z16 DMMA) and the TC kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/s2c12_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c12_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2c12_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s2c12_smoke.log
timeout 1200 python bench.py --gate-out gpurun_out/s2c12_gate.jsonl > gpurun_out/s2c12_bench.json 2> gpurun_out/s2c12_bench.err
echo "bench rc=$?" >> gpurun_out/s2c12_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bulk_kernel|gather_kernel|scale_kernel|direct_kernel' -c 40 --csv \
  --log-file gpurun_out/s2c12_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/s2c12_launch_bench.log 2>&1
PROF_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bulk_kernel' -o /tmp/ncu/bench -f \
  python tools/prof_list.py "z16NNgen d16NNgen s16NNgen s10NNgen" > gpurun_out/s2c12_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/bench.ncu-rep > gpurun_out/s2c12_ncu_bench.json 2>> gpurun_out/s2c12_ncu.log
PROF_REPS=1 timeout 600 ncu --set full --clock-control none -k regex:'tc_kernel' -o /tmp/ncu/tc -f \
  python tools/prof_list.py "s64NNgen s64NNb0 c32NNgen c32NNb0 s57NNgen" 100000 > gpurun_out/s2c12_ncu_tc.log 2>&1
python tools/ncu_summary.py /tmp/ncu/tc.ncu-rep > gpurun_out/s2c12_ncu_tc.json 2>> gpurun_out/s2c12_ncu_tc.log
tail -4 gpurun_out/s2c12_pytest.log; tail -3 gpurun_out/s2c12_smoke.log; tail -2 gpurun_out/s2c12_bench.err; head -c 300 gpurun_out/s2c12_bench.json; du -sh gpurun_out
