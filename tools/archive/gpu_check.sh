set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "sweep or nonsquare or integer" > gpurun_out/pytest1.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest1.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/bench1.log
