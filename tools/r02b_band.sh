#!/bin/bash
# K2 band-size sweep (tuning build, DGDIFF_K2_BAND caps the rows per band):
# the launcher aims at ~8 items per SM; c5 (64 sources) has few items per band
for band in 0 64 32 16; do
  for cfg in "--config c5 --sources 64 --degree 2 --nsteps 8" "--config c5 --sources 64 --degree 3 --nsteps 2" "--config c5 --sources 64 --degree 2 --element 1 --nsteps 8" "--nsteps 2"; do
    echo "band=$band $cfg: $(DGDIFF_TUNING_LIB=1 DGDIFF_K2_BAND=$band DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py $cfg --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
done
