#!/bin/bash
# quads with item neighbour buffers: parity tests, then c5 stage times
timeout 900 python -m pytest tests -m gpu -q -x -k "quad or Q1 or Q2 or element or subpixel or absorb or window" > gpurun_out/quad_pytest.log 2>&1; tail -3 gpurun_out/quad_pytest.log
for d in 2 1; do
  echo "Q$d: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --degree $d --element 1 --nsteps 8 --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  echo "Q$d fp32: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --precision 32 --degree $d --element 1 --nsteps 8 --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
done
