#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k3d" > gpurun_out/pytest_k3d.log 2>&1
timeout 600 python tools/try_pair.py 0,5 > gpurun_out/try_pair.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_golden.py -m gpu -q > gpurun_out/pytest_golden.log 2>&1
tail -3 gpurun_out/pytest_k3d.log; cat gpurun_out/try_pair.log; tail -3 gpurun_out/pytest_golden.log
