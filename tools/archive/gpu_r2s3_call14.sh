#!/bin/bash
# Round 2 (session 3), call 14: sizes 17-32, all types, N/N, both epilogues, the default plan
# (the NEXT-4 table of the docs) plus S=2 x 16 KB for s (a beta = 0 rule candidate).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c14
S=17,18,19,20,21,22,23,24,25,26,27,28,29,30,31,32
timeout 1500 python tools/tune_big.py --kinds s --sizes $S --tunings 0:0,2:16 --bytes 6e8 --out gpurun_out/${P}_big.jsonl > gpurun_out/${P}_big.log 2>&1
timeout 1500 python tools/tune_big.py --kinds dcz --sizes $S --tunings 0:0 --bytes 6e8 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
tail -2 gpurun_out/${P}_big.log; du -sh gpurun_out
