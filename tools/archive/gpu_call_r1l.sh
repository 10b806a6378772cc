cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 900 python -m pytest tests -m gpu -q -x -k "nonsquare or swizzled" > gpurun_out/pt_l.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_l.log
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16,12x7x16 --layout strided --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ns_swz_on3.jsonl > /dev/null 2>> gpurun_out/nsswz.err; echo ns rc=$?
