# TRA instances' own searched mappings (libtxgemm_tra.so, all ON) vs shipped: cur / tra / cur / tra.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in cur1 tra cur2 tra2; do
  case $v in tra*) export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_tra.so;; *) unset TXGEMM_LIB;; esac
  timeout 1200 python tools/sweep.py --sizes 2-16 --ops TN,TT,CN,CT,CC,TC --reps 20 --graph --out gpurun_out/tra_$v.jsonl > /dev/null 2>> gpurun_out/tra.err; echo $v rc=$?
done
tail -2 gpurun_out/tra.err
