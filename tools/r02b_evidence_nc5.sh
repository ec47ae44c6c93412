#!/bin/bash
# Round-2 (second session) evidence on one GPU, outputs under gpurun_out/ev2_*:
# bench lines (K2 default with cpu_baseline, K3d, fp32, P2, reference arm),
# the ncu launch list of the bench, ncu --set full of one K2 step (DRAM
# traffic per launch); no c5 run (see r02_c5_full_runs.jsonl).
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/ev2_bench.json 2> gpurun_out/ev2_bench.err
timeout 600 python bench.py --steps 5 --warmup 3 --temporal-steps 5 --no-cpu-baseline > gpurun_out/ev2_bench_k3d.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --precision 32 --no-cpu-baseline > gpurun_out/ev2_bench_fp32.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --degree 2 --no-cpu-baseline > gpurun_out/ev2_bench_p2.json 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ev2_ref.json 2> gpurun_out/ev2_ref.err
for f in ev2_bench ev2_bench_k3d ev2_bench_fp32 ev2_bench_p2 ev2_ref; do tail -1 gpurun_out/$f.json | cut -c1-200; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/ev2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev2_ncu_launch.log 2>&1
timeout 300 python tools/prof_stage.py --precision 64 --degree 1 --nsteps 2 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage_ring -s 3 -c 3 -o gpurun_out/ev2_full_p1_fp64 \
  python tools/prof_stage.py --precision 64 --degree 1 --nsteps 2 --reps 1 > gpurun_out/ev2_ncu_full.log 2>&1
tail -1 gpurun_out/ev2_ncu_full.log
