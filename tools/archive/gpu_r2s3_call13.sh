#!/bin/bash
# Round 2 (session 3), call 13: DMMA rule beyond 16 (z 17-25 and d 33-47 on CUDA cores) --
# parity tests beyond 16 / non-square / DMMA, default-plan sweep of the affected sizes.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c13
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "beyond or odd_large or nonsquare or dmma" > gpurun_out/${P}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
timeout 900 python tools/tune_big.py --kinds zd --sizes 17,20,24,25,28,32 --tunings 0:0 --out gpurun_out/${P}_big.jsonl > gpurun_out/${P}_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds d --sizes 36,40,44,48,56,64 --tunings 0:0 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
tail -3 gpurun_out/${P}_pytest.log; tail -2 gpurun_out/${P}_big.log; du -sh gpurun_out
