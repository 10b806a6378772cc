cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "beyond_16" > gpurun_out/pt_y.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_y.log
