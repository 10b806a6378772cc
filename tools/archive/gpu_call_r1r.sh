# Two-CTA tile shrink for runtime-specialised bulk plans: on / off / on / off.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 900 python -m pytest tests -m gpu -q -x -k "nonsquare or beyond or swizzled" > gpurun_out/pt_r.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_r.log
for v in on1 off1 on2 off2; do
  case $v in off*) export TX_PLAN_2CTA=0;; *) unset TX_PLAN_2CTA;; esac
  timeout 900 python tools/sweep.py --sizes 17-32 --batch 300000 --ops NN,TN --reps 6 --out gpurun_out/p2_big_$v.jsonl > /dev/null 2>> gpurun_out/p2.err; echo big $v rc=$?
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16,12x7x16 --layout strided --ops NN,TT --reps 10 --out gpurun_out/p2_ns_$v.jsonl > /dev/null 2>> gpurun_out/p2.err; echo ns $v rc=$?
done
tail -2 gpurun_out/p2.err
