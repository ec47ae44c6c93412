#!/bin/bash
mkdir -p gpurun_out
for ser in 0 1; do
  export DGDIFF_TUNING_LIB=1 DGDIFF_RING_SERIAL=$ser
  echo "serial=$ser"
  python tools/prof_stage.py --precision 64 --degree 1 --nsteps 4 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c4 P1 fp64 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  python tools/prof_stage.py --precision 32 --degree 1 --nsteps 4 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c4 P1 fp32 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  python tools/prof_stage.py --config c5 --sources 64 --degree 2 --nsteps 8 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c5 P2 fp64 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  python tools/prof_stage.py --config c5 --sources 64 --degree 3 --nsteps 4 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c5 P3 fp64 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  python tools/prof_stage.py --config c5 --sources 64 --degree 2 --element 1 --nsteps 8 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c5 Q2 fp64 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  python tools/prof_stage.py --config c5 --sources 64 --degree 1 --element 1 --nsteps 8 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c5 Q1 fp64 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  python bench.py --steps 3 --warmup 3 --windows 1 --no-cpu-baseline --k3d-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  c4 windows bench ms/step %.1f frac %.3f'%(d['ms_per_step'], d['roofline']['frac']))"
done
