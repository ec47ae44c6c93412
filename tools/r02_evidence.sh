#!/bin/bash
# Round-2 evidence on one GPU (outputs under gpurun_out/): the GPU suite,
# smoke, bench lines (K2 default, K3d, fp32, P2, reference arm), the ncu launch
# list of the bench, and ncu --set full captures of the stage kernels (DRAM
# traffic per launch for profiles/stage_traffic.json)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.log 2>&1; tail -2 gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; tail -1 gpurun_out/ev_smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --steps 5 --warmup 3 --temporal-steps 5 --no-cpu-baseline > gpurun_out/ev_bench_k3d.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --precision 32 --no-cpu-baseline > gpurun_out/ev_bench_fp32.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --degree 2 --no-cpu-baseline > gpurun_out/ev_bench_p2.json 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
for f in ev_bench ev_bench_k3d ev_bench_fp32 ev_bench_p2 ev_ref; do tail -1 gpurun_out/$f.json | cut -c1-160; done
# ncu: launch list of the bench (plain run above exited), then full captures
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
for v in "64 1 0" "32 1 0" "64 2 0" "64 1 5" "32 1 5"; do
  set -- $v
  if [ "$3" = "5" ]; then K=k_stage_pair; S=1; C=1; else K=k_stage_ring; S=3; C=3; fi
  timeout 300 python tools/prof_stage.py --precision $1 --degree $2 --tb $3 --nsteps 2 --reps 1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:$K -s $S -c $C -o gpurun_out/ev_full_p$2_fp$1_ts$3 \
    python tools/prof_stage.py --precision $1 --degree $2 --tb $3 --nsteps 2 --reps 1 > gpurun_out/ev_ncu_full_p$2_fp$1_ts$3.log 2>&1
  tail -1 gpurun_out/ev_ncu_full_p$2_fp$1_ts$3.log
done
