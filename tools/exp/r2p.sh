timeout 1200 python -m pytest -q -x tests -m gpu > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
timeout 600 python bench.py --config C > /tmp/c.log 2>&1; tail -1 /tmp/c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C tok/s', d['tokens_per_s'], 'e2e', d['e2e']['tokens_per_s'])"
