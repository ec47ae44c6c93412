#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1907_06191_b200/csrc -o /tmp/pixel_bench tools/pixel_bench.cu && /tmp/pixel_bench > gpurun_out/pixel_bench.log 2>&1
cat gpurun_out/pixel_bench.log
