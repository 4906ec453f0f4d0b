timeout 1200 python -m pytest -q -x tests -m gpu 2>&1 | tail -2
for pdl in 1 0; do PKV_PDL=$pdl timeout 600 python bench.py --config C --stream-steps 1024 > gpurun_out/b6_C_$pdl.log 2>&1; tail -1 gpurun_out/b6_C_$pdl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('PDL $pdl C tok/s', d['tokens_per_s'], d['us_per_token'], 'e2e', d['e2e']['tokens_per_s'])"; done
