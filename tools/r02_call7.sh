#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_bw tools/tma_bw.cu && /tmp/tma_bw > gpurun_out/tma_bw.json 2>&1
for r in 0,0 40,0 70,0; do
 echo "K2 diag ring $r: $(DGDIFF_TUNING_LIB=1 DGDIFF_K2_DIAG=1 DGDIFF_RING=$r PAIR_CASES=c4_p1_fp64 timeout 300 python tools/try_pair.py 0 2>&1 | tail -1)" >> gpurun_out/k2_diag.log
 echo "K2 ring $r: $(DGDIFF_TUNING_LIB=1 DGDIFF_RING=$r PAIR_CASES=c4_p1_fp64 timeout 300 python tools/try_pair.py 0 2>&1 | tail -1)" >> gpurun_out/k2_diag.log
done
cat gpurun_out/tma_bw.json gpurun_out/k2_diag.log
