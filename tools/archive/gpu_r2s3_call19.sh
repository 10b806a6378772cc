#!/bin/bash
# Round 2 (session 3), call 19: end-of-session validation of the committed tree -- full GPU suite,
# smoke, the default bench line, the reference arm, ncu --set full of the bench kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
P=s3c19
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/${P}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${P}_smoke.log
timeout 1200 python bench.py --gate-out gpurun_out/${P}_gate.jsonl > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
echo "bench rc=$?" >> gpurun_out/${P}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
echo "ref rc=$?" >> gpurun_out/${P}_bench_ref.err
PROF_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bulk_kernel' -o /tmp/ncu/bench -f \
  python tools/prof_list.py "z16NNgen d16NNgen s16NNgen s10NNgen" > gpurun_out/${P}_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/bench.ncu-rep > gpurun_out/${P}_ncu_bench.json 2>> gpurun_out/${P}_ncu.log
tail -3 gpurun_out/${P}_pytest.log; tail -3 gpurun_out/${P}_smoke.log; tail -1 gpurun_out/${P}_bench.err; head -c 300 gpurun_out/${P}_bench.json; head -c 300 gpurun_out/${P}_bench_ref.json; du -sh gpurun_out
