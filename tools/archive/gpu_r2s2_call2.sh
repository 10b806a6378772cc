#!/bin/bash
# Round 2 (session 2), call 2: tcgen05 probe, tensor-core kernel parity, DMMA A/B (d/z n <= 16)
# and TC A/B (s/c beyond 16) with the gate protocol, ncu of the TC kernel.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/tc_probe.py > gpurun_out/s2c2_tcprobe.json 2> gpurun_out/s2c2_tcprobe.err
echo "probe rc=$?" >> gpurun_out/s2c2_tcprobe.err
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > gpurun_out/s2c2_pytest_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c2_pytest_tc.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "beyond_16" > gpurun_out/s2c2_pytest_big.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c2_pytest_big.log
for r in 1 2; do
  for d in 1 0; do
    TX_DMMA=$d timeout 600 python tools/gate_run.py --kinds dz --sizes 1-16 --out gpurun_out/s2c2_dmma${d}_r$r.jsonl 2>> gpurun_out/s2c2_gate.err
  done
done
for r in 1 2; do
  for t in 1 0; do
    TX_TC=$t timeout 900 python tools/gate_run.py --kinds s --sizes 17,20,24,28,32,36,40,48,56,64 --ops NN,TT,TN --out gpurun_out/s2c2_tcs${t}_r$r.jsonl 2>> gpurun_out/s2c2_gate.err
    TX_TC=$t timeout 900 python tools/gate_run.py --kinds c --sizes 17,18,20,22,24,26,28,30,32 --ops NN,CT,TC --out gpurun_out/s2c2_tcc${t}_r$r.jsonl 2>> gpurun_out/s2c2_gate.err
  done
done
TX_TC=1 PROF_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'tc_kernel' -o /tmp/ncu/tc -f \
  python tools/prof_list.py "s64NNgen s64NNb0 c32NNgen c32NNb0 s32NNgen c24NNgen" 100000 > gpurun_out/s2c2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s2c2_ncu.log
python tools/ncu_summary.py /tmp/ncu/tc.ncu-rep > gpurun_out/s2c2_ncu_tc.json 2>> gpurun_out/s2c2_ncu.log
cp /tmp/ncu/tc.ncu-rep gpurun_out/s2c2_tc.ncu-rep
cat gpurun_out/s2c2_tcprobe.json | head -50; tail -15 gpurun_out/s2c2_pytest_tc.log; tail -3 gpurun_out/s2c2_pytest_big.log; tail -12 gpurun_out/s2c2_gate.err; du -sh gpurun_out
