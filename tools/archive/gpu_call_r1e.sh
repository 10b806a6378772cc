# Final-table sweeps: every square instance (graph-timed, clocks sampled), configs[3] shapes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python tools/sweep.py --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 20 --graph --out gpurun_out/sweep_v7.jsonl > /dev/null 2> gpurun_out/sweep_v7.err; echo sweep rc=$?
tail -2 gpurun_out/sweep_v7.err
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3 --layout ptr --ops NN,TT,CC --reps 10 --out gpurun_out/ptr_v7.jsonl > /dev/null 2>> gpurun_out/sweep_v7.err; echo ptr rc=$?
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3 --layout strided --ops NN,TT,CC --reps 10 --out gpurun_out/ns_v7.jsonl > /dev/null 2>> gpurun_out/sweep_v7.err; echo ns rc=$?
bash tools/gpu_bench_all.sh
