timeout 300 python -m pytest tests -m gpu -q -x -k "store or fused_default or smoke" 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(d.get('compressor'))" || tail -20 gpurun_out/b.log
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "prefill/" --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/comp.csv 2>&1
grep '^"' gpurun_out/comp.csv | python -c "
import sys,csv
r=list(csv.reader(sys.stdin))
h=r[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
from collections import defaultdict
d=defaultdict(float); n=defaultdict(int)
for x in r[1:]:
  if len(x)>vi: d[x[ki][:50]]+=float(x[vi].replace(',','')); n[x[ki][:50]]+=1
for k in d: print(n[k], round(d[k]/1e3/n[k],1), k)
"
