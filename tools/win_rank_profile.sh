for v in "1 0" "8 0"; do
  set -- $v
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wrp_$1.csv python tools/win_rank_profile.py $1 $2 > /dev/null 2>&1
  python - "$1" <<'PY'
import csv,sys,collections
rows=list(csv.reader(open(f"gpurun_out/wrp_{sys.argv[1]}.csv")))
h=rows[0]; i=h.index("Kernel Name"); v=h.index("Metric Value")
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    if len(r)<=v: continue
    try: t=float(r[v].replace(',',''))
    except: continue
    k=r[i].split('(')[0][:60]; agg[k][0]+=1; agg[k][1]+=t
tot=sum(x[1] for x in agg.values())
print("R", sys.argv[1], "total ms", round(tot/1e6,1))
for k,(n,t) in sorted(agg.items(), key=lambda kv:-kv[1][1])[:8]: print(f"  {k:60s} {n:6d} {t/1e6:9.1f} ms")
PY
done
