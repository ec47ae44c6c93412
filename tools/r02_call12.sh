#!/bin/bash
mkdir -p gpurun_out
for d in 3 9 8; do for w in 0 7,4; do
  echo "diag $d warps $w: $(DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_WARPS=$w DGDIFF_PAIR_DIAG=$d PAIR_CASES=c4_p1_fp64 timeout 300 python tools/try_pair.py 5 2>&1 | tail -1)" >> gpurun_out/pair_diag2.log
done; done
cat gpurun_out/pair_diag2.log
