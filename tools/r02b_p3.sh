#!/bin/bash
# P3 column-form kernel: parity tests, then c5 stage times (column form vs the
# round-1 immediates in the tuning build compiled with -DDGDIFF_P3_IMM)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "p3 or P3 or subpixel or absorb" > gpurun_out/p3_pytest.log 2>&1; tail -3 gpurun_out/p3_pytest.log
for lib in 0 1; do
  for prec in 64 32; do
    echo "tuning_lib(imm)=$lib prec=$prec"
    DGDIFF_TUNING_LIB=$lib timeout 300 python tools/prof_stage.py --config c5 --sources 64 --degree 3 --precision $prec --nsteps 4 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['runs'][-1]; print('  c5 P3 stage ms %.3f GB/s %.0f'%(r['stage_ms'], r['gbs']))"
  done
done
