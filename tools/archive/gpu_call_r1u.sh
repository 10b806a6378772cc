# Host-buffer entry: pipeline chunk size sweep (bench e2e line).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
for mb in 32 64 128 512; do
  export TX_HOSTIO_CHUNK_MB=$mb
  timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/e2e_$mb_$r.log 2>&1
  echo "mb $mb r $r $(tail -1 gpurun_out/e2e_$mb_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"], d["value"])')"
done
done
