cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "square_sweep_all_ops and (z-10 or 10-z)" > gpurun_out/pt_za.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_za.log
timeout 600 python -m pytest tests -m gpu -q -x -k "integer or batch_edges" > gpurun_out/pt_za2.log 2>&1; echo pytest2 rc=$?; tail -2 gpurun_out/pt_za2.log
