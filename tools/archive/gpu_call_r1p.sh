cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "square_sweep or integer or fullsize" > gpurun_out/pt_p.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_p.log
timeout 900 python tools/sweep.py --kinds cz --sizes 13-16 --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 20 --out gpurun_out/pc_merged.jsonl > /dev/null 2>> gpurun_out/pc.err; echo merged rc=$?
