#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k3d" 2>&1 | tail -1
for w in 0 6,4; do for pf in 0 3 6 12 24; do
  echo "warps $w pf $pf: $(DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_WARPS=$w DGDIFF_PAIR_PF=$pf PAIR_CASES=c4_p1_fp64,c4_p1_fp32 timeout 300 python tools/try_pair.py 5 2>&1 | tail -2 | tr '\n' ' ')"
done; done
