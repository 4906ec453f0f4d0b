python -m pytest -q -x tests/test_gpu_single_pass.py 2>&1 | tail -2
for c in B E D; do timeout 300 python tools/exp/kbench.py s a --cfg $c --reps 10 2>&1 | tail -2; done
PKV_ATTN_INLINE_MERGE=1 timeout 300 python tools/exp/kbench.py s --cfg B --reps 10 2>&1 | tail -1
timeout 600 python bench.py --config C --stream-steps 512 --steps 64 --warmup 3 > gpurun_out/b3_C.log 2>&1; tail -1 gpurun_out/b3_C.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C tok/s', d['tokens_per_s'], d['us_per_token'], 'e2e', d['e2e']['tokens_per_s'])"
