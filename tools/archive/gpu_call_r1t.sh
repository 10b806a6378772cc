cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 900 python -m pytest tests -m gpu -q -x -k "odd_sizes or pointer or swizzled or nonsquare or beyond" > gpurun_out/pt_t.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_t.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "odd_sizes and 37" > gpurun_out/san_u16.log 2>&1; echo memcheck rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_u16.log | tail -2
timeout 900 python tools/sweep.py --shapes 5x7x3,7x7x7,3x3x3 --layout ptr --ops NN,TT --reps 10 --out gpurun_out/u16_on.jsonl > /dev/null 2>> gpurun_out/u16.err; echo u16 rc=$?
tail -2 gpurun_out/u16.err
