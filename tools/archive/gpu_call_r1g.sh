# BSWG: swizzled-gather tests, A/B on pointer arrays.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 1200 python -m pytest tests -m gpu -q -x -k "swizzled or pointer or padded or nonsquare or jit or device" > gpurun_out/pt_bsw.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_bsw.log
for v in on off; do
  if [ $v = off ]; then export TX_JIT_ASW=0; fi
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --layout ptr --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ptr_bswg_$v.jsonl > /dev/null 2>> gpurun_out/bswg.err; echo ptr $v rc=$?
done
tail -2 gpurun_out/bswg.err
