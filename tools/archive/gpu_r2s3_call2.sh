#!/bin/bash
# Round 2 (session 3), call 2: pointer-array kernel A/B (bulk_ptr vs 16-byte gather, pipeline
# settings, DMMA on/off) on configs[3] shapes + 16x16x16, and the tcgen05-vs-CUDA-core A/B
# behind the tensor-core default rule (tc_rule).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c2
SH=16x16x16,16x3x16,8x16x4,1x16x16,4x6x16,16x16x1
T=0:0,2:16,3:16,4:16,2:32,3:32,2:64
timeout 900 python tools/ptr_ab.py --shapes $SH --tunings $T --strided --out gpurun_out/${P}_ptr_ab.jsonl > gpurun_out/${P}_ptr_ab.log 2>&1
echo "ab1 rc=$?" >> gpurun_out/${P}_ptr_ab.log
TX_PTR_BULK_MIN=1000000 timeout 900 python tools/ptr_ab.py --shapes 16x16x16,16x3x16,8x16x4 --tunings 0:0 --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
echo "ab2 rc=$?" >> gpurun_out/${P}_ptr_ab.log
TX_PTR_BULK_MIN=64 timeout 900 python tools/ptr_ab.py --shapes 1x16x16,4x6x16,16x16x1 --tunings 0:0,2:16,3:32 --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
echo "ab3 rc=$?" >> gpurun_out/${P}_ptr_ab.log
TX_DMMA=0 timeout 900 python tools/ptr_ab.py --kinds dz --shapes $SH --tunings 0:0,2:16,3:32 --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
echo "ab4 rc=$?" >> gpurun_out/${P}_ptr_ab.log
for tc in 0 1; do
  TX_TC=$tc timeout 900 python tools/gate_run.py --kinds s --sizes 17,24,32,40,48,56,57,64 --ops NN --out gpurun_out/${P}_tc_ab_s_$tc.jsonl > gpurun_out/${P}_tc_ab_s_$tc.log 2>&1
  TX_TC=$tc timeout 900 python tools/gate_run.py --kinds c --sizes 13,16,20,24,28,29,32 --ops NN,CT --out gpurun_out/${P}_tc_ab_c_$tc.jsonl > gpurun_out/${P}_tc_ab_c_$tc.log 2>&1
done
tail -2 gpurun_out/${P}_ptr_ab.log; grep -c . gpurun_out/${P}_ptr_ab.jsonl; tail -1 gpurun_out/${P}_tc_ab_c_1.log; du -sh gpurun_out
