# ASWG (swizzled A placement in gather kernels): full GPU tests, A/B on pointer arrays.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_all.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_all.log
for v in on off; do
  if [ $v = off ]; then export TX_JIT_ASW=0; fi
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --layout ptr --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ptr_aswg_$v.jsonl > /dev/null 2>> gpurun_out/aswg.err; echo ptr $v rc=$?
done
tail -2 gpurun_out/aswg.err
