# Power-capped re-search, third batch (s/d n = 3-8, c/z n = 3-4): cur, pc, cur, pc (graph-timed).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in cur1 pc cur2 pc2; do
  case $v in pc*) export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_pc.so;; *) unset TXGEMM_LIB;; esac
  timeout 900 python tools/sweep.py --kinds sd --sizes 3-8 --ops NN,NT,TN,TT --reps 20 --graph --out gpurun_out/pcc_sd_$v.jsonl > /dev/null 2>> gpurun_out/pcc.err; echo sd $v rc=$?
  timeout 900 python tools/sweep.py --kinds cz --sizes 3-4 --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 20 --graph --out gpurun_out/pcc_cz_$v.jsonl > /dev/null 2>> gpurun_out/pcc.err; echo cz $v rc=$?
done
tail -2 gpurun_out/pcc.err
