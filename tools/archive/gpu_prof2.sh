cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bulk_kernel|gather_kernel|scale_kernel" -c 24 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 2400 python tools/sweep.py --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 10 --out gpurun_out/sweep_ops.jsonl > /dev/null 2> gpurun_out/sweep.err; echo sweep rc=$?
tail -2 gpurun_out/sweep.err
