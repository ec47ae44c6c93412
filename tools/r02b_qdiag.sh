#!/bin/bash
# Q2/Q1/P1/P2/P3 ring kernel: full compute vs streaming the rows without compute
# (DGDIFF_K2_DIAG=1, tuning build): is the row pipeline (TMA issue) the bound?
for d in 0 1; do
  for cfg in "--degree 2 --element 1 --nsteps 8" "--degree 1 --element 1 --nsteps 8" "--degree 2 --nsteps 8" "--degree 3 --precision 32 --nsteps 4"; do
    echo "diag=$d $cfg: $(DGDIFF_TUNING_LIB=1 DGDIFF_K2_DIAG=$d DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 $cfg --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
  echo "diag=$d c4 P1: $(DGDIFF_TUNING_LIB=1 DGDIFF_K2_DIAG=$d DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --nsteps 2 --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
done
