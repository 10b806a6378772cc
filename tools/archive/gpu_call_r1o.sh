# Square c/z n = 13-16: current table vs the power-capped re-search (libtxgemm_pc.so), cur-pc-cur.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in cur1 pc cur2 pc2; do
  case $v in pc*) export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_pc.so;; *) unset TXGEMM_LIB;; esac
  timeout 900 python tools/sweep.py --kinds cz --sizes 13-16 --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 20 --out gpurun_out/pc_$v.jsonl > /dev/null 2>> gpurun_out/pc.err; echo $v rc=$?
done
tail -2 gpurun_out/pc.err
