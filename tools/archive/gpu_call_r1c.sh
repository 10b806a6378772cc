cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep.py --sizes 1-6 --graph --reps 40 --out gpurun_out/small_graph.jsonl > /dev/null 2> gpurun_out/small_graph.err; echo small rc=$?
for c in "s 1 NN 1" "s 2 NN 1" "c 16 TN 1" "c 16 TN 0" "z 16 TN 1" "d 16 TN 1"; do
  set -- $c
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 2 -c 1 -o gpurun_out/prof_$1$2$3_$4 python tools/prof_case.py $1 $2 $3 $4 > /dev/null 2>&1; echo "$c rc=$?"
done
export TX_JIT_CACHE=/tmp/jit_model_$$
timeout 900 python tools/sweep.py --sizes 17-32 --batch 300000 --reps 6 --ops TT,TN --kinds sd --out gpurun_out/ab_bigT_model.jsonl > /dev/null 2>>gpurun_out/ab.err
timeout 900 python tools/sweep.py --sizes 17-32 --batch 300000 --reps 6 --ops CC,CN --kinds cz --out gpurun_out/ab_bigC_model.jsonl > /dev/null 2>>gpurun_out/ab.err
export TX_JIT_MAP=heuristic; export TX_JIT_CACHE=/tmp/jit_heur_$$
timeout 900 python tools/sweep.py --sizes 17-32 --batch 300000 --reps 6 --ops TT,TN --kinds sd --out gpurun_out/ab_bigT_heuristic.jsonl > /dev/null 2>>gpurun_out/ab.err
timeout 900 python tools/sweep.py --sizes 17-32 --batch 300000 --reps 6 --ops CC,CN --kinds cz --out gpurun_out/ab_bigC_heuristic.jsonl > /dev/null 2>>gpurun_out/ab.err
echo ab done
