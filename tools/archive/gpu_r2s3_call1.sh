#!/bin/bash
# Round 2 (session 3), call 1: re-entry check of the restored tree (smoke, default bench line with
# gate), the pointer-array pattern roof over configs[3] shapes, and ncu --set full of every
# gate-failing strided instance plus the pointer-array worst cases.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
P=s3c1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 1200 python bench.py --gate-out gpurun_out/${P}_gate.jsonl > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
echo "bench rc=$?" >> gpurun_out/${P}_bench.err
timeout 900 python tools/ptr_roof.py --out gpurun_out/${P}_ptr_roof.jsonl > gpurun_out/${P}_ptr_roof.log 2>&1
echo "roof rc=$?" >> gpurun_out/${P}_ptr_roof.log
PROF_REPS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'bulk_kernel|direct_kernel' -o /tmp/ncu/gate -f \
  python tools/prof_list.py "c13CCb0 c13NNb0 c14CCb0 c16CNb0 c7NCb0 c9NNb0 c5NNb0 c5NNgen s3NTb0 s10NNb0 s11NTb0 z10CTb0 z9TCb0 s1NNb0 s1NNgen c1NNb0 d1NNb0" > gpurun_out/${P}_ncu_gate.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${P}_ncu_gate.log
python tools/ncu_summary.py /tmp/ncu/gate.ncu-rep > gpurun_out/${P}_ncu_gate.json 2>> gpurun_out/${P}_ncu_gate.log
ncu -i /tmp/ncu/gate.ncu-rep --page details --csv > gpurun_out/${P}_ncu_gate_details.csv 2>/dev/null; gzip -f gpurun_out/${P}_ncu_gate_details.csv
for c in "s 5 7 3 NN 1" "z 4 6 16 NN 1" "s 16 3 16 NN 1" "s 4 6 16 NN 1"; do
  set -- $c
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:'gather|bulk_ptr' -c 2 -o /tmp/ncu/ptr_$1_$2_$3_$4 -f \
    python tools/prof_ptr_case.py $c >> gpurun_out/${P}_ncu_ptr.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/ptr_$1_$2_$3_$4.ncu-rep > gpurun_out/${P}_ncu_ptr_$1_$2_$3_$4.json 2>> gpurun_out/${P}_ncu_ptr.log
done
tail -3 gpurun_out/${P}_smoke.log; tail -2 gpurun_out/${P}_bench.err; head -c 400 gpurun_out/${P}_bench.json; tail -2 gpurun_out/${P}_ptr_roof.log; tail -2 gpurun_out/${P}_ncu_gate.log; du -sh gpurun_out
