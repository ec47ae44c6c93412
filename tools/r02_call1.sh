#!/bin/bash
# round-2 GPU call 1: host info, FMA peaks, GPU suite (minus the golden tests
# whose fixtures are still being generated), compute-sanitizer on the pipelines
mkdir -p gpurun_out
{ nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fma_peak tools/fma_peak.cu && /tmp/fma_peak > gpurun_out/fma_peak.json 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "not golden" > gpurun_out/pytest_gpu.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_case.py ring > gpurun_out/san_ring_$t.log 2>&1
  echo "exit $?" >> gpurun_out/san_ring_$t.log
done
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_case.py wave > gpurun_out/san_wave_$t.log 2>&1
  echo "exit $?" >> gpurun_out/san_wave_$t.log
done
tail -3 gpurun_out/pytest_gpu.log
