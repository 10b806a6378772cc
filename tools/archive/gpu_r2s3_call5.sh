#!/bin/bash
# Round 2 (session 3), call 5: per-(type, n) ncu evidence for the gate: every type x n = 1..16,
# N/N, beta = 0 and general, 10^6 pairs, one captured launch each (DRAM bytes, shared-memory
# wavefronts / conflicts, pipes, issue, clock) -> tools/ncu_table.py.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c5
SPECS="$(cat tools/ncu_gate_specs.txt)"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
PROF_REPS=1 timeout 1800 ncu --metrics $M --clock-control none -k regex:'bulk_kernel|direct_kernel' --csv --log-file gpurun_out/${P}_ncu_gate.csv \
  python tools/prof_list.py "$SPECS" > gpurun_out/${P}_ncu_gate.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${P}_ncu_gate.log
python tools/ncu_table.py gpurun_out/${P}_ncu_gate.csv "$SPECS" > gpurun_out/${P}_ncu_table.jsonl 2>> gpurun_out/${P}_ncu_gate.log
gzip -f gpurun_out/${P}_ncu_gate.csv
tail -2 gpurun_out/${P}_ncu_gate.log; wc -l gpurun_out/${P}_ncu_table.jsonl; du -sh gpurun_out
