# Multi-rank bench path (2 ranks on one GPU, gloo) and a final bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --dist-backend gloo --no-cpu > gpurun_out/bench_mr.log 2>&1; echo mr rc=$?
tail -1 gpurun_out/bench_mr.log | cut -c1-300
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 1 --impl reference > gpurun_out/bench_ref_mr.log 2>&1; echo refmr rc=$?
tail -1 gpurun_out/bench_ref_mr.log | cut -c1-200
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_default.log | cut -c1-200
