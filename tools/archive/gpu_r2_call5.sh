#!/bin/bash
# Round 2, call 5: DMMA parity + A/B sweep (d/z all ops, 10^6 pairs), ncu of z16 with DMMA.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ring.py -m gpu -q -x -p no:cacheprovider \
  -k "dmma or square_sweep or integer or ring_square or transposed_a or pointer_array_equals" > gpurun_out/r2c5_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c5_pytest.log
for d in 1 0 1 0; do
  TX_DMMA=$d timeout 600 python tools/sweep.py --kinds dz --sizes 1-16 --ops NN,NT,TN,TT,CN,NC,CC,TC,CT --graph \
    --out gpurun_out/r2c5_dmma${d}_$RANDOM.jsonl > /dev/null 2>> gpurun_out/r2c5_sweep.err
done
PROF_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'bulk_kernel' -o /tmp/ncu/dmma -f \
  python tools/prof_list.py "z16NNgen d16NNgen z16TNb0 z13NNb0" > gpurun_out/r2c5_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu/dmma.ncu-rep > gpurun_out/r2c5_ncu_dmma.json 2>> gpurun_out/r2c5_ncu.log
tail -3 gpurun_out/r2c5_pytest.log; du -sh gpurun_out
