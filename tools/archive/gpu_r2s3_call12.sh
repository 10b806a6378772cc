#!/bin/bash
# Round 2 (session 3), call 12: d / z beyond 16 -- DMMA on/off x pipeline settings; s17 beta = 0.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c12
for dm in 1 0; do
  TX_DMMA=$dm timeout 900 python tools/tune_big.py --kinds z --sizes 17,20,24,28,32 --tunings 0:0,2:16,2:32,2:64 --out gpurun_out/${P}_dmma$dm.jsonl > gpurun_out/${P}.log 2>&1
  TX_DMMA=$dm timeout 900 python tools/tune_big.py --kinds d --sizes 17,24,40,48,56,64 --tunings 0:0,2:16,2:32,2:64 --out gpurun_out/${P}_dmma$dm.jsonl >> gpurun_out/${P}.log 2>&1
done
timeout 600 python tools/tune_big.py --kinds s --sizes 17,19,21 --tunings 0:0,2:16,2:32,2:64,3:16 --out gpurun_out/${P}_s17.jsonl >> gpurun_out/${P}.log 2>&1
tail -2 gpurun_out/${P}.log; du -sh gpurun_out
