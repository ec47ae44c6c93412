"""Hottest SASS lines of one kernel from `ncu --page source --csv --print-source sass`:
  python tools/sass_hot.py src.csv <kernel-substring> [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want, N = sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
b = next(b for b in blocks if want in b["name"])
hdr, data = b["rows"][0], b["rows"][1:]
ix = {h: i for i, h in enumerate(hdr)}
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(float(r[ix[h]] or 0) for r in data) for h in stall_cols}
print("total samples", tot)
print("by reason:", sorted(((round(v / tot * 100, 1), k) for k, v in agg.items() if v), reverse=True)[:10])
data.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:N]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((float(r[ix[h]] or 0), h) for h in stall_cols), reverse=True)[:2]
    print(f"{s / tot * 100:5.2f}% {r[ix['Address']]:>6} {r[ix['Source']][:70]:70} {[(h[6:], int(v)) for v, h in top if v]}")
