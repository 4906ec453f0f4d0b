#!/bin/bash
# GPU-side quick check: parity tests + one bench line summary
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 800 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; c=d.get('cublas',{})
print('value', d['value'], 'K us', k['fused_k_us'], 'V us', k['fused_v_us'], 'K GB/s phys', k['fused_k_gbs_physical'], 'V', k['fused_v_gbs_physical'], 'cublas', c.get('k_us'), c.get('v_us'), 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
