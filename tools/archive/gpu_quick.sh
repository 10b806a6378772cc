# Quick GPU loop: parity (subset or all), bench, launch list + full ncu of the bench kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SEL=${SEL:-}
timeout 1200 python -m pytest tests -m gpu -q -x $SEL > gpurun_out/pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest.log
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -2 gpurun_out/bench.log | cut -c1-1500
if [ -n "$PROF" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bulk_kernel|gather_kernel|scale_kernel" -c 20 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 4 -c 2 -o gpurun_out/prof_bench python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
fi
