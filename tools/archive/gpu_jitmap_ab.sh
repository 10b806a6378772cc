cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jit_model_$$
timeout 1500 python -m pytest tests -m gpu -q -x -k "nonsquare or jit or pointer or beyond or fixed or device or config4" > gpurun_out/pt.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pt.log
for mode in model heuristic; do
  if [ $mode = heuristic ]; then export TX_JIT_MAP=heuristic; export TX_JIT_CACHE=/tmp/jit_heur_$$; fi
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3 --layout strided --ops NN,TT --reps 8 --out gpurun_out/ab_ns_$mode.jsonl > /dev/null 2>>gpurun_out/ab.err
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3 --layout ptr --ops NN,TT --reps 8 --out gpurun_out/ab_ptr_$mode.jsonl > /dev/null 2>>gpurun_out/ab.err
  timeout 900 python tools/sweep.py --sizes 17-32 --batch 300000 --reps 6 --out gpurun_out/ab_big_$mode.jsonl > /dev/null 2>>gpurun_out/ab.err
  echo $mode done
done
tail -3 gpurun_out/ab.err
