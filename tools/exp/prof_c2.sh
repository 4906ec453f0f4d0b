mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --config C --stream-steps 200 --steps 64 --warmup 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_C2.csv')) if r]
hdr=next(r for r in rows if r[0]=='ID'); ik=hdr.index('Kernel Name'); iv=hdr.index('Metric Value')
ks=[(r[ik][:50], float(r[iv].replace(',',''))) for r in rows if r[0].isdigit()]
tail=ks[-40*3*20:]
c=collections.defaultdict(list)
for k,v in tail: c[k].append(v)
for k,v in sorted(c.items(), key=lambda kv:-sum(kv[1])): print(len(v), round(sum(v)/len(v)/1e3,2), k)
PY
