cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/sweep.py --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 10 --out gpurun_out/sweep_ops_${TAG}.jsonl > /dev/null 2> gpurun_out/sweep.err; echo sweep rc=$?
tail -2 gpurun_out/sweep.err
