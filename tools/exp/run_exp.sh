#!/bin/bash
# A/B timing of library variants (experiments; results are not parity-checked)
for v in base "$@"; do
  if [ $v != base ]; then cp tools/exp/lib$v.so paper_2512_24449_b200/libpackkv_b200.so; fi
  timeout 90 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cublas > /tmp/exp_$v.log 2>&1
  tail -1 /tmp/exp_$v.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$v', d['kernels']['fused_k_us'], d['kernels']['fused_v_us'])
except Exception: print('$v FAILED')"
done
