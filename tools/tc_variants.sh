#!/bin/bash
# Build measurement variants of the tensor-core kernel (tools/tc_trace.cu) and time them
# (tools/tc_trace.py --so): default, no suspend hint, and with one stage of the pipeline
# removed (transform / MMA / epilogue) to see which one bounds a shape.  Needs a GPU.
cd "$(dirname "$0")/.."
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include -I paper_1304_7053_b200/csrc -shared -Xcompiler -fPIC"
declare -A V=( [base]="" [nohint]="-DTC_SUSPEND_NS=0" [notr]="-DTC_EXP_NOTRANSFORM" [nomma]="-DTC_EXP_NOMMA" [noepi]="-DTC_EXP_NOEPI" )
for v in "${!V[@]}"; do $NV ${V[$v]} -o /tmp/tcv_$v.so tools/tc_trace.cu & done; wait
for c in "c 32 32 32 gen" "c 32 32 32 b0" "s 64 64 64 gen" "s 48 48 48 b0" "c 24 24 24 b0" "c 20 20 20 gen"; do
  for v in base nohint notr nomma noepi; do
    python tools/tc_trace.py $c 100000 --so /tmp/tcv_$v.so --quiet
  done
done
