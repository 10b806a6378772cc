#!/bin/bash
# Round-2 GPU validation: full -m gpu suite with per-test durations, then smoke.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.free,clocks.sm --format=csv > gpurun_out/r2_nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=60 -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
tail -5 gpurun_out/r2_pytest.log; tail -3 gpurun_out/r2_smoke.log
