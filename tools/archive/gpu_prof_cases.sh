cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "$@"; do
  set -- $c
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 2 -c 1 -o gpurun_out/prof_$1$2$3_$4 python tools/prof_case.py $1 $2 $3 $4 > /dev/null 2>&1; echo "$c rc=$?"
done
