#!/bin/bash
# Round 2 (session 3), call 6: FFMA2 (sm_100 packed fp32 FMA) complex MAC vs the scalar FFMA chain
# (build_noffma2, -DTX_NO_FFMA2): interleaved gate sweeps over c (all n, all op pairs, both
# epilogues), bitwise check on integer inputs through the c parity tests, ncu of c13/c16 b0;
# pointer arrays with transposed A: bulk_ptr vs the 16-byte gather (ASWG); then call 5 (per-type ncu).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
P=s3c6
NOFF=$PWD/paper_1304_7053_b200/libtxgemm_noffma2.so
export TX_JIT_CACHE=/tmp/txjit_$$
for r in 1 2; do
  timeout 600 python tools/gate_run.py --kinds c --tag ffma2_$r --out gpurun_out/${P}_gate_ffma2_$r.jsonl >> gpurun_out/${P}_gate.log 2>&1
  TXGEMM_LIB=$NOFF timeout 600 python tools/gate_run.py --kinds c --tag ffma_$r --out gpurun_out/${P}_gate_ffma_$r.jsonl >> gpurun_out/${P}_gate.log 2>&1
done
timeout 1500 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_ring.py > gpurun_out/${P}_pytest_c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest_c.log
PROF_REPS=1 timeout 600 ncu --set full --clock-control none -k regex:'bulk_kernel' -o /tmp/ncu/ff -f \
  python tools/prof_list.py "c13NNb0 c13CCb0 c16CNb0 c9NNb0 c16NNgen" > gpurun_out/${P}_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/ff.ncu-rep > gpurun_out/${P}_ncu_ffma2.json 2>> gpurun_out/${P}_ncu.log
timeout 600 python tools/ptr_ab.py --kinds zdc --shapes 16x3x16,8x16x4,16x16x16 --ops NN,TT,CN --tag default --out gpurun_out/${P}_ptr_ab.jsonl > gpurun_out/${P}_ptr_ab.log 2>&1
TX_PTR_BULK_MIN=1000000 timeout 600 python tools/ptr_ab.py --kinds zdc --shapes 16x3x16,8x16x4,16x16x16 --ops NN,TT,CN --tag gather16 --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
bash tools/gpu_r2s3_call5.sh
tail -2 gpurun_out/${P}_gate.log; tail -2 gpurun_out/${P}_pytest_c.log; du -sh gpurun_out
