cd $GRAFT_REPO_ROOT
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3 --layout ptr --ops NN,TT --reps 10 --out gpurun_out/sweep_ptr.jsonl > /dev/null 2>gpurun_out/sweep_ptr.err; echo ptr rc=$?
timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3 --layout strided --ops NN,TT --reps 10 --out gpurun_out/sweep_ns.jsonl > /dev/null 2>>gpurun_out/sweep_ptr.err; echo ns rc=$?
tail -3 gpurun_out/sweep_ptr.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --dist-backend gloo --no-cpu > gpurun_out/bench_mr.log 2>&1; echo mr rc=$?
tail -2 gpurun_out/bench_mr.log | cut -c1-400
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 1 --impl reference > gpurun_out/bench_ref_mr.log 2>&1; echo refmr rc=$?
tail -1 gpurun_out/bench_ref_mr.log | cut -c1-300
