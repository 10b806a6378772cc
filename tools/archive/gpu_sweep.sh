cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | cut -c1-900
timeout 1500 python tools/sweep.py --out gpurun_out/sweep_nn.jsonl > /dev/null 2> gpurun_out/sweep.err; echo sweep rc=$?
tail -3 gpurun_out/sweep.err
