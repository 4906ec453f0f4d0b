mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_single_pass.py -q -x 2>&1 | tail -2
for c in B E; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-cublas > gpurun_out/b2_$c.log 2>&1; tail -1 gpurun_out/b2_$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'K', d['kernels']['fused_k_us'], 'V', d['kernels']['fused_v_us'], 'attn', d['attention'], 'e2e', d['e2e']['ms_per_step'])"; done
timeout 600 python bench.py --config C --stream-steps 1024 --steps 64 --warmup 3 > gpurun_out/b2_C.log 2>&1; tail -1 gpurun_out/b2_C.log | cut -c 1-200; tail -1 gpurun_out/b2_C.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C tok/s', d['tokens_per_s'], d['us_per_token'], 'e2e', d['e2e'])"
