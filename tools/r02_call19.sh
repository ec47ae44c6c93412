#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build19.log 2>&1
python tools/try_p3.py
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "p3 or absorb or degenerate or subpixel" 2>&1 | tail -2
