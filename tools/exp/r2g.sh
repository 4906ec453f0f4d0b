timeout 900 python -m pytest -q -x tests/test_gpu_fastpath.py tests/test_gpu_parity.py -k "graphed or decode or append" 2>&1 | tail -3
python tools/exp/dbg_append.py 2 2>&1 | tail -2
timeout 600 python bench.py --config C --stream-steps 512 --steps 64 --warmup 3 > gpurun_out/b4_C.log 2>&1; tail -1 gpurun_out/b4_C.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C tok/s', d['tokens_per_s'], d['us_per_token'], 'e2e', d['e2e']['tokens_per_s'])"
