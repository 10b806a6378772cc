#!/bin/bash
# Round 2 (session 3), call 3: decoupled ring (empty mbarriers + rotated warp items) vs the
# round-1 per-tile __syncthreads ring (build_nodec, -DTX_NO_DEC): interleaved gate sweeps and
# pointer-array A/B; n = 1, 2 size-matched roof; then the full GPU suite on the new library.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c3
NODEC=$PWD/paper_1304_7053_b200/libtxgemm_nodec.so
export TX_JIT_CACHE=/tmp/txjit_$$
for r in 1 2; do
  timeout 600 python tools/gate_run.py --tag dec$r --out gpurun_out/${P}_gate_dec.jsonl >> gpurun_out/${P}_gate.log 2>&1
  TXGEMM_LIB=$NODEC timeout 600 python tools/gate_run.py --tag nodec$r --out gpurun_out/${P}_gate_nodec.jsonl >> gpurun_out/${P}_gate.log 2>&1
done
echo "gate done" >> gpurun_out/${P}_gate.log
SH=16x16x16,16x3x16,8x16x4,1x16x16,4x6x16,16x16x1,5x7x3
timeout 900 python tools/ptr_ab.py --shapes $SH --tunings 0:0,2:16,2:32,3:32 --tag dec --out gpurun_out/${P}_ptr_ab.jsonl > gpurun_out/${P}_ptr_ab.log 2>&1
TXGEMM_LIB=$NODEC timeout 900 python tools/ptr_ab.py --shapes $SH --tunings 0:0,2:16,2:32,3:32 --tag nodec --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
TX_PTR_BULK_MIN=1000000 timeout 900 python tools/ptr_ab.py --shapes 16x16x16,16x3x16,8x16x4 --tunings 0:0 --tag dec_gather16 --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
TX_PTR_BULK_MIN=64 timeout 900 python tools/ptr_ab.py --shapes 1x16x16,4x6x16,16x16x1 --tunings 0:0,2:16,2:32 --tag dec_bulk64 --out gpurun_out/${P}_ptr_ab.jsonl >> gpurun_out/${P}_ptr_ab.log 2>&1
echo "ptr done" >> gpurun_out/${P}_ptr_ab.log
timeout 300 python tools/n1_roof.py --out gpurun_out/${P}_n1_roof.jsonl > gpurun_out/${P}_n1_roof.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/${P}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
tail -3 gpurun_out/${P}_gate.log; tail -2 gpurun_out/${P}_ptr_ab.log; tail -3 gpurun_out/${P}_n1_roof.log; tail -4 gpurun_out/${P}_pytest.log; du -sh gpurun_out
