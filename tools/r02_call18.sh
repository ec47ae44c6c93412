#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build18.log 2>&1
timeout 1500 python tools/dg_mc_refine.py --factors 1,2,4 --degrees 1 > gpurun_out/dg_mc_refine.jsonl 2> gpurun_out/dg_mc_refine.err
timeout 900 python tools/dg_mc_refine.py --factors 1,2 --degrees 2 2>> gpurun_out/dg_mc_refine.err | grep '"dg"' >> gpurun_out/dg_mc_refine.jsonl
cat gpurun_out/dg_mc_refine.jsonl; tail -3 gpurun_out/dg_mc_refine.err
