#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k3d" > gpurun_out/pytest_k3d.log 2>&1; tail -1 gpurun_out/pytest_k3d.log
timeout 600 python tools/try_pair.py 0,5 > gpurun_out/try_pair.log 2>&1; cat gpurun_out/try_pair.log
for w in 0 6,5 8,4; do for d in 0 9; do
  echo "W6 warps $w diag $d: $(DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_WARPS=$w DGDIFF_PAIR_DIAG=$d PAIR_CASES=c4_p1_fp64,c4_p1_fp32 timeout 300 python tools/try_pair.py 5 2>&1 | tail -2 | tr '\n' ' ')" >> gpurun_out/pair_w6.log
done; done
cat gpurun_out/pair_w6.log
