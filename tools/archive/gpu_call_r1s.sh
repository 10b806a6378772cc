cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
for v in on1 off1 on2; do
  case $v in off*) export TX_PLAN_2CTA=0;; *) unset TX_PLAN_2CTA;; esac
  for s in 19 23 25 26 27 28 32; do
    timeout 300 python tools/sweep.py --sizes $s --batch 300000 --ops NN,TN --reps 6 --out gpurun_out/p3_big_${v}_$s.jsonl > /dev/null 2>> gpurun_out/p3.err
  done
  echo big $v
  timeout 900 python tools/sweep.py --shapes 16x3x16,12x7x16 --layout strided --ops NN,TT --reps 10 --out gpurun_out/p3_ns_$v.jsonl > /dev/null 2>> gpurun_out/p3.err; echo ns $v rc=$?
done
tail -2 gpurun_out/p3.err
