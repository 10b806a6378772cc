#!/bin/bash
# Round 2, call 6: full GPU suite (DMMA + sizes to 64), DMMA pipeline autotune, DMMA A/B on pointer arrays.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=25 > gpurun_out/r2c6_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c6_pytest.log
TX_DMMA=1 timeout 1200 python tools/autotune.py --kinds dz --sizes 5-16 --out gpurun_out/r2c6_mma_autotune.jsonl > /dev/null 2> gpurun_out/r2c6_autotune.err
for d in 1 0; do
  TX_DMMA=$d timeout 600 python tools/ptr_roof.py --kinds dz --shapes 16x16x16,8x16x4,16x3x16,1x16x16,4x6x16,16x16x1,13x13x13 \
    --out gpurun_out/r2c6_ptr_dmma$d.jsonl > /dev/null 2>> gpurun_out/r2c6_ptr.err
done
tail -30 gpurun_out/r2c6_pytest.log | grep -v "^[0-9.]*s call" ; du -sh gpurun_out
