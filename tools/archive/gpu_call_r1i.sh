# JIT bulk swizzles (TMA tensor A/B tiles for non-square strided shapes): tests, sanitizers, A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_all2.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_all2.log
python tools/sanitize_case.py > /dev/null 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san2_$tool.log 2>&1; echo $tool rc=$?; tail -1 gpurun_out/san2_$tool.log
done
timeout 600 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_case.py --uninit-c > gpurun_out/san2_initcheck.log 2>&1; echo initcheck rc=$?; tail -1 gpurun_out/san2_initcheck.log
for v in on off; do
  if [ $v = off ]; then export TX_JIT_ASW=0; fi
  timeout 900 python tools/sweep.py --shapes 8x16x4,16x3x16,1x16x16,16x16x1,5x7x3,4x6x16,12x7x16 --layout strided --ops NN,TT,TN,CC,CN --reps 10 --out gpurun_out/ns_swz_$v.jsonl > /dev/null 2>> gpurun_out/nsswz.err; echo ns $v rc=$?
done
tail -2 gpurun_out/nsswz.err
