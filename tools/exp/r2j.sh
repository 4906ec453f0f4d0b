timeout 900 python -m pytest -q -x tests/test_gpu_fastpath.py tests/test_gpu_parity.py tests/test_gpu_single_pass.py -k "graphed or decode or append or flush or single or store" 2>&1 | tail -2
python tools/exp/dbg_append.py 2 2>&1 | tail -1
timeout 600 python bench.py --config C > gpurun_out/b5_C.log 2>&1; tail -1 gpurun_out/b5_C.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C tok/s', d['tokens_per_s'], d['us_per_token'], 'e2e', d['e2e']['tokens_per_s'])"
