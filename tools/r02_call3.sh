#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1
python tools/prof_pair.py 5 > gpurun_out/prof_pair_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stage_pair -s 1 -c 1 -o gpurun_out/pair_c4 python tools/prof_pair.py 5 > gpurun_out/ncu_pair.log 2>&1
tail -5 gpurun_out/ncu_pair.log
