# ASW (TMA tensor-copy A tiles): parity, sanitizers, A/B sweep against a no-ASW build, ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "transposed_a_tensor or (square_sweep_all_ops and 16)" > gpurun_out/pt_asw.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_asw.log
python tools/sanitize_case.py > /dev/null 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san_$tool.log 2>&1; echo $tool rc=$?; tail -1 gpurun_out/san_$tool.log
done
timeout 600 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_case.py --uninit-c > gpurun_out/san_initcheck.log 2>&1; echo initcheck rc=$?; tail -1 gpurun_out/san_initcheck.log
for v in asw noasw; do
  if [ $v = noasw ]; then export TXGEMM_LIB=$GRAFT_REPO_ROOT/paper_1304_7053_b200/libtxgemm_noasw.so; fi
  timeout 900 python tools/sweep.py --kinds dcz --sizes 16 --ops NN,NT,TN,TT,CN,CT,TC,CC,NC --reps 20 --out gpurun_out/asw_$v.jsonl > /dev/null 2>> gpurun_out/asw.err; echo sweep $v rc=$?
done
unset TXGEMM_LIB
for c in "d 16 TN 1" "z 16 TN 1" "c 16 TN 1" "z 16 TN 0"; do
  set -- $c
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 2 -c 1 -o gpurun_out/prof_asw_$1$2$3_$4 python tools/prof_case.py $1 $2 $3 $4 > /dev/null 2>&1; echo "$c rc=$?"
done
