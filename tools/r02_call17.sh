#!/bin/bash
mkdir -p gpurun_out
echo "new (constant-bank P3):"; python tools/try_p3.py
echo "old (literals, tuning lib built from HEAD):"; DGDIFF_TUNING_LIB=1 python tools/try_p3.py
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "p3" 2>&1 | tail -2
