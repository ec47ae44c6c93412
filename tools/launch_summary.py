"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel counts, totals and shares.  python tools/launch_summary.py in.csv out.json"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ik, iv, iu = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
per = collections.defaultdict(list)
unit = None
for r in data:
    if len(r) <= iv:
        continue
    try:
        v = float(r[iv].replace(',', ''))
    except ValueError:
        continue
    unit = r[iu]
    per[r[ik].split('(')[0].replace('void ', '')].append(v)
tot = sum(sum(v) for v in per.values())
out = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); "
                 "command: python bench.py --steps 3 --warmup 3 --no-cpu-baseline",
       "unit": unit, "total_launches": sum(len(v) for v in per.values()), "kernels": {}}
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    out["kernels"][k] = {"launches": len(v), "total": sum(v), "mean": sum(v) / len(v), "share": sum(v) / tot}
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, d in out["kernels"].items():
    print(f"{d['share']:.4f} {d['launches']:4d} {d['mean']/1e6:9.3f} ms  {k}")
