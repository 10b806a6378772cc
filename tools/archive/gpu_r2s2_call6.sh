#!/bin/bash
# Round 2 (session 2), call 6: M=64 TMEM layout probe, TC kernel v3 (M=64, windowed stages) parity,
# odd-large-size fix, full GPU suite, TC trace + A/B, ncu summary of the TC kernel.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/tc_probe.py > gpurun_out/s2c6_tcprobe.json 2> gpurun_out/s2c6_tcprobe.err
python -c "import json;d=json.load(open('gpurun_out/s2c6_tcprobe.json'));print('m64 rule', d.get('m64_lane_of_row_rule_16x4'), d.get('m64_exact_16x4_rule'))"
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/s2c6_pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c6_pytest_tc.log
tail -3 gpurun_out/s2c6_pytest_tc.log
for c in "c 32 32 32 gen" "s 64 64 64 gen" "c 24 24 24 b0" "s 40 40 40 gen"; do
  echo "== $c" >> gpurun_out/s2c6_trace.txt
  timeout 300 python tools/tc_trace.py $c >> gpurun_out/s2c6_trace.txt 2>&1
done
grep steady gpurun_out/s2c6_trace.txt
for t in 1 0; do
  TX_TC=$t timeout 1200 python tools/gate_run.py --kinds s --sizes 17-64 --ops NN,TT --out gpurun_out/s2c6_tcs${t}.jsonl 2>> gpurun_out/s2c6_gate.err
  TX_TC=$t timeout 900 python tools/gate_run.py --kinds c --sizes 9-32 --ops NN,CT,TC --out gpurun_out/s2c6_tcc${t}.jsonl 2>> gpurun_out/s2c6_gate.err
done
TX_TC=1 PROF_REPS=1 timeout 600 ncu --set full --clock-control none -k regex:'tc_kernel' -o /tmp/ncu/tc -f \
  python tools/prof_list.py "s64NNgen c32NNgen c32NNb0 s40NNgen c24NNb0" 100000 > gpurun_out/s2c6_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/tc.ncu-rep > gpurun_out/s2c6_ncu_tc.json 2>> gpurun_out/s2c6_ncu.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=20 > gpurun_out/s2c6_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c6_pytest.log
tail -4 gpurun_out/s2c6_pytest.log; grep -c "" gpurun_out/s2c6_gate.err; du -sh gpurun_out
