#!/bin/bash
# Round 2 (session 3), call 16: per-size plan override for square s with beta = 0 beyond 16 --
# parity tests beyond 16 and the s 17-32 sweep (default plan, twice).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
P=s3c16
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "beyond or odd_large" > gpurun_out/${P}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
for r in 1 2; do
timeout 900 python tools/tune_big.py --kinds s --sizes 17,18,19,20,21,22,23,24,25,26,27,28,29,30,31,32 --tunings 0:0 --bytes 6e8 --out gpurun_out/${P}_s_$r.jsonl > gpurun_out/${P}_s.log 2>&1
done
tail -3 gpurun_out/${P}_pytest.log; du -sh gpurun_out
