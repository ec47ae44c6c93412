#!/bin/bash
mkdir -p gpurun_out
for d in 0 1 2 3 4; do for w in 6,5 8,6; do
  echo "diag $d warps $w: $(DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_WARPS=$w DGDIFF_PAIR_DIAG=$d DGDIFF_PAIR_PF=0 PAIR_CASES=c4_p1_fp64 timeout 300 python tools/try_pair.py 5 2>&1 | tail -1)" >> gpurun_out/pair_diag.log
done; done
cat gpurun_out/pair_diag.log
