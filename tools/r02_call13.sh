#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k3d" > gpurun_out/pytest_k3d.log 2>&1; tail -1 gpurun_out/pytest_k3d.log
for pf in 0 2 4 8 12; do for w in 0 7,4; do for d in 0 9; do
  echo "pf $pf warps $w diag $d: $(DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_PF=$pf DGDIFF_PAIR_WARPS=$w DGDIFF_PAIR_DIAG=$d PAIR_CASES=c4_p1_fp64,c4_p1_fp32 timeout 300 python tools/try_pair.py 5 2>&1 | tail -2 | tr '\n' ' ')" >> gpurun_out/pair_pf.log
done; done; done
cat gpurun_out/pair_pf.log
