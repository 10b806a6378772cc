#!/bin/bash
# Round 2 (session 3), call 17: pipeline settings for c / z / d beyond 16 (both epilogues).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c17
S=17,18,19,20,21,22,23,24,25,26,27,28
timeout 1500 python tools/tune_big.py --kinds cz --sizes $S --tunings 0:0,2:16,2:32,2:64 --bytes 6e8 --out gpurun_out/${P}_big.jsonl > gpurun_out/${P}_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds d --sizes $S --tunings 0:0,2:16,2:32,2:64 --bytes 6e8 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
tail -1 gpurun_out/${P}_big.log; du -sh gpurun_out
