timeout 1200 python -m pytest -q -x tests -m gpu 2>&1 | tail -1
for pdl in 1 0; do echo "PDL=$pdl"; PKV_PDL=$pdl timeout 300 python tools/exp/kbench.py a k v --cfg B --reps 10 2>&1 | tail -3; done
PKV_PDL=1 timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-cublas > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('PDL1 e2e', d['e2e']['ms_per_step'], d['attention'])"
PKV_PDL=0 timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-cublas > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('PDL0 e2e', d['e2e']['ms_per_step'], d['attention'])"
