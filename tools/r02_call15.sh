#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_bw tools/tma_bw.cu && /tmp/tma_bw > gpurun_out/tma_bw2.json 2>&1
sed -n '/rows/,$p' gpurun_out/tma_bw2.json
