#!/bin/bash
mkdir -p gpurun_out
python tools/prof_pair.py 5 > gpurun_out/prof_pair_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stage_pair -s 1 -c 1 -o gpurun_out/pair_c4d python tools/prof_pair.py 5 > gpurun_out/ncu_pair.log 2>&1
tail -2 gpurun_out/ncu_pair.log
