cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_all.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_default.log | cut -c1-200
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bulk_kernel|gather_kernel|scale_kernel" -c 24 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
