#!/bin/bash
# Re-entry check after the container restore: GPU suite, smoke, bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c1_pytest.log 2>&1; tail -3 gpurun_out/c1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1; tail -1 gpurun_out/c1_smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
tail -1 gpurun_out/c1_bench.json | cut -c1-400
