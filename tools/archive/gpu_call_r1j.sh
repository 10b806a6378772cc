cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 900 python -m pytest tests -m gpu -q -x -k "nonsquare or swizzled or transposed_a or square_sweep" > gpurun_out/pt_j.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_j.log
timeout 900 python tools/sweep.py --shapes 16x3x16,1x16x16,4x6x16,12x7x16 --layout strided --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ns_swz_on2.jsonl > /dev/null 2>> gpurun_out/nsswz.err; echo ns rc=$?
timeout 900 python tools/sweep.py --kinds dcz --sizes 16 --ops NN,NT,TN,TT,CN,CT,TC,CC,NC --reps 20 --out gpurun_out/sq16_recheck.jsonl > /dev/null 2>> gpurun_out/nsswz.err; echo sq rc=$?
