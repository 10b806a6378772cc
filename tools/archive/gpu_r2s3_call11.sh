#!/bin/bash
# Round 2 (session 3), call 11: the sizes-beyond-16 general plan rule (two 32 KB stages) --
# parity tests beyond 16 and the default-plan sweep.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c11
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "beyond or odd_large or nonsquare" > gpurun_out/${P}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
timeout 900 python tools/tune_big.py --kinds s --sizes 17,24,32,40,48,56,64 --tunings 0:0 --out gpurun_out/${P}_big.jsonl > gpurun_out/${P}_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds cdz --sizes 17,20,24,28,32 --tunings 0:0 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds d --sizes 40,48,56,64 --tunings 0:0 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
tail -3 gpurun_out/${P}_pytest.log; tail -2 gpurun_out/${P}_big.log; du -sh gpurun_out
