# Balanced contiguous partition of the bulk kernel vs round-robin tiles (libtxgemm_rr.so).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 1500 python -m pytest tests -m gpu -q -x -k "square_sweep or batch_edges or deterministic or transposed_a or fixed or device or fullsize" > gpurun_out/pt_n.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_n.log
for r in 1 2 3; do
  for v in new rr; do
    if [ $v = rr ]; then export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_rr.so; else unset TXGEMM_LIB; fi
    timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/bench_$v$r.log 2>&1
    echo "$v $r $(tail -1 gpurun_out/bench_$v$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["gbps"], d["roofline"]["frac"], d["roofline"]["per_size_gbps"], d["clocks"]["sm_mhz"])')"
  done
done
for v in new rr; do
  if [ $v = rr ]; then export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_rr.so; else unset TXGEMM_LIB; fi
  timeout 600 python tools/sweep.py --sizes 8-16 --batch 100000 --graph --reps 40 --out gpurun_out/part_$v.jsonl > /dev/null 2>> gpurun_out/part.err; echo sweep $v rc=$?
done
