# Power-capped re-search, second batch (s/d n = 9-16, c/z n = 5-12): cur, pc, cur, pc.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in cur1 pc cur2 pc2; do
  case $v in pc*) export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_pc.so;; *) unset TXGEMM_LIB;; esac
  timeout 900 python tools/sweep.py --kinds sd --sizes 9-16 --ops NN,NT,TN,TT --reps 20 --out gpurun_out/pcb_sd_$v.jsonl > /dev/null 2>> gpurun_out/pcb.err; echo sd $v rc=$?
  timeout 900 python tools/sweep.py --kinds cz --sizes 5-12 --ops NN,NT,TN,TT,NC,CN,CC,TC,CT --reps 20 --out gpurun_out/pcb_cz_$v.jsonl > /dev/null 2>> gpurun_out/pcb.err; echo cz $v rc=$?
done
tail -2 gpurun_out/pcb.err
