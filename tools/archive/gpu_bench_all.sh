cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cfg2 cfg1 cfg5d cfg5z; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
  tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','gbps','hbm_frac']}, d['roofline']['frac'], d['roofline']['achieved'], (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
done
