# Gather ring depth: GS = 3 (shipped) vs 4 (libtxgemm_gs4.so), pointer arrays, cur / gs4 / cur / gs4.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in cur1 gs4 cur2 gs42; do
  case $v in gs4*) export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_gs4.so;; *) unset TXGEMM_LIB;; esac
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16 --layout ptr --ops NN,TT,CN --reps 10 --out gpurun_out/gs_$v.jsonl > /dev/null 2>> gpurun_out/gs.err; echo $v rc=$?
done
tail -2 gpurun_out/gs.err
