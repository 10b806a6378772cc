cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sanitize_case.py > /dev/null 2>&1   # warm the JIT disk cache outside the sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san_$tool.log 2>&1; echo $tool rc=$?; tail -2 gpurun_out/san_$tool.log
done
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_case.py --uninit-c > gpurun_out/san_initcheck.log 2>&1; echo initcheck rc=$?; tail -2 gpurun_out/san_initcheck.log
