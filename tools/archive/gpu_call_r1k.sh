cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TX_JIT_CACHE=/tmp/jitc_$$
for v in on off; do
  if [ $v = off ]; then export TX_JIT_ASW=0; fi
  python tools/prof_ns_case.py z 16 3 16 TT 0 > /dev/null 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 2 -c 1 -o gpurun_out/prof_ns_z16x3x16_TT_0_$v python tools/prof_ns_case.py z 16 3 16 TT 0 > gpurun_out/prof_ns_$v.log 2>&1; echo "$v rc=$?"
done
