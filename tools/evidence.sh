# Round evidence on one GPU: bench line, ncu launch list, ncu --set full of one
# SSP-RK3 step (launches 7-9 = stages 1-3 of the first timed step... after warm-up).
set -e
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_line.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench_line.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -s 6 -c 3 -o gpurun_out/stage_full \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
