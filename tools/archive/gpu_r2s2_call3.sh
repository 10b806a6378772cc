#!/bin/bash
# Round 2 (session 2), call 3: the measurements of call 2 again (its output exceeded the
# 64 MiB merge limit): tcgen05 probe, DMMA A/B (d/z n <= 16), TC A/B (s 17-64, c 9-32),
# ncu summary of the TC kernel (no .ncu-rep copied back).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/tc_probe.py > gpurun_out/s2c3_tcprobe.json 2> gpurun_out/s2c3_tcprobe.err
for r in 1 2; do
  for d in 1 0; do
    TX_DMMA=$d timeout 600 python tools/gate_run.py --kinds dz --sizes 1-16 --out gpurun_out/s2c3_dmma${d}_r$r.jsonl 2>> gpurun_out/s2c3_gate.err
  done
done
for r in 1 2; do
  for t in 1 0; do
    TX_TC=$t timeout 1200 python tools/gate_run.py --kinds s --sizes 17-64 --ops NN,TT --out gpurun_out/s2c3_tcs${t}_r$r.jsonl 2>> gpurun_out/s2c3_gate.err
    TX_TC=$t timeout 900 python tools/gate_run.py --kinds c --sizes 9-32 --ops NN,CT,TC --out gpurun_out/s2c3_tcc${t}_r$r.jsonl 2>> gpurun_out/s2c3_gate.err
  done
done
TX_TC=1 PROF_REPS=1 timeout 600 ncu --set full --clock-control none -k regex:'tc_kernel' -o /tmp/ncu/tc -f \
  python tools/prof_list.py "s64NNgen s64NNb0 c32NNgen c32NNb0 s32NNgen c24NNgen c13NNb0" 100000 > gpurun_out/s2c3_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s2c3_ncu.log
python tools/ncu_summary.py /tmp/ncu/tc.ncu-rep > gpurun_out/s2c3_ncu_tc.json 2>> gpurun_out/s2c3_ncu.log
tail -12 gpurun_out/s2c3_gate.err; du -sh gpurun_out
