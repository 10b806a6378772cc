# Full GPU test suite, launch list and one full ncu capture of the bench's kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_all.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
