#!/bin/bash
# Round 2 (session 3), call 18: per-size plan table beyond 16 -- parity beyond 16, then the
# default-plan sweep of d / c / z 17-28 and s 17-32 (to compare with the tuning sweep).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c18
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "beyond or odd_large or nonsquare" > gpurun_out/${P}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
timeout 900 python tools/tune_big.py --kinds dcz --sizes 17,18,19,20,21,22,23,24,25,26,27,28 --tunings 0:0 --bytes 6e8 --out gpurun_out/${P}_big.jsonl > gpurun_out/${P}_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds s --sizes 17,18,19,20,21,22,23,24,25,26,27,28,29,30,31,32 --tunings 0:0 --bytes 6e8 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
timeout 900 python tools/tune_big.py --kinds dcz --sizes 29,30,31,32 --tunings 0:0 --bytes 6e8 --out gpurun_out/${P}_big.jsonl >> gpurun_out/${P}_big.log 2>&1
tail -3 gpurun_out/${P}_pytest.log; du -sh gpurun_out
