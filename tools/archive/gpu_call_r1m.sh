# Gather ring stage-size target sweep (pointer arrays, configs[3] shapes).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
for kb in 16 8 4 32; do
  export TX_GATHER_KB=$kb
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --layout ptr --ops NN,TT,CN --reps 10 --out gpurun_out/ptr_kb$kb.jsonl > /dev/null 2>> gpurun_out/kb.err; echo kb $kb rc=$?
done
tail -2 gpurun_out/kb.err
