cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_default.log | cut -c1-160
