cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "s 5 7 3 NN 1" "z 4 6 16 NN 1" "d 16 16 1 NN 1"; do
  set -- $c
  python tools/prof_ptr_case.py $1 $2 $3 $4 $5 $6 > /dev/null 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 2 -c 1 -o gpurun_out/prof_ptr_$1$2x$3x$4_$5_$6 python tools/prof_ptr_case.py $1 $2 $3 $4 $5 $6 > /dev/null 2>&1; echo "$c rc=$?"
done
