#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build16.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ts0.json 2> gpurun_out/bench_ts0.err
python bench.py --steps 5 --warmup 3 --temporal-steps 5 --no-cpu-baseline > gpurun_out/bench_ts5.json 2> gpurun_out/bench_ts5.err
python bench.py --steps 5 --warmup 3 --precision 32 --no-cpu-baseline > gpurun_out/bench_fp32_ts0.json 2>&1
python bench.py --steps 5 --warmup 3 --precision 32 --temporal-steps 5 --no-cpu-baseline > gpurun_out/bench_fp32_ts5.json 2>&1
python bench.py --steps 3 --warmup 3 --degree 2 --no-cpu-baseline > gpurun_out/bench_p2.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
for f in bench_ts0 bench_ts5 bench_fp32_ts0 bench_fp32_ts5 bench_p2 bench_ref; do python -c "
import json,sys
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
r=d.get('roofline',{})
print('$f', '%.4g'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'frac', r.get('frac'), r.get('kernel'), 'share', r.get('share_of_step'), d.get('cpu_baseline',{}).get('one_core'), d.get('cpu_baseline',{}).get('all_cores'), d.get('clocks'))
"; done
