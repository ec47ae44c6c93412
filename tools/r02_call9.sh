#!/bin/bash
mkdir -p gpurun_out
export DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_DIAG=3
python tools/prof_pair.py 5 > gpurun_out/prof_pair_diag_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stage_pair -s 1 -c 1 -o gpurun_out/pair_diag3 python tools/prof_pair.py 5 > gpurun_out/ncu_pair_diag.log 2>&1
tail -2 gpurun_out/ncu_pair_diag.log
