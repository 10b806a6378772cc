# Round-end checkpoint: smoke, all GPU tests, bench + reference arm, launch list, ncu of the
# bench kernels, final graph-timed all-ops sweep and configs[3] sweeps.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bulk_kernel|gather_kernel|scale_kernel" -c 24 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 3000 python tools/sweep.py --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 20 --graph --out gpurun_out/sweep_v8.jsonl > /dev/null 2> gpurun_out/sweep_v8.err; echo sweep rc=$?
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --layout ptr --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ptr_v8.jsonl > /dev/null 2>> gpurun_out/sweep_v8.err; echo ptr rc=$?
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16,12x7x16 --layout strided --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ns_v8.jsonl > /dev/null 2>> gpurun_out/sweep_v8.err; echo ns rc=$?
bash tools/gpu_bench_all.sh
