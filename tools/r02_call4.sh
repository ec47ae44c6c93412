#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k3d" > gpurun_out/pytest_k3d.log 2>&1
timeout 600 python tools/try_pair.py 0,5 > gpurun_out/try_pair.log 2>&1
python tools/prof_pair.py 5 > gpurun_out/prof_pair_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stage_pair -s 1 -c 1 -o gpurun_out/pair_c4b python tools/prof_pair.py 5 > gpurun_out/ncu_pair.log 2>&1
tail -3 gpurun_out/pytest_k3d.log; cat gpurun_out/try_pair.log; tail -2 gpurun_out/ncu_pair.log
