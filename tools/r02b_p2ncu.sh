#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stage_ring -s 3 -c 2 -o gpurun_out/p2 \
  python tools/prof_stage.py --config c5 --sources 64 --degree 2 --precision 64 --nsteps 2 --reps 1 > gpurun_out/p2_ncu.log 2>&1
tail -1 gpurun_out/p2_ncu.log
