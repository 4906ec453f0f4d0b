cp paper_2512_24449_b200/libpackkv_b200.so /tmp/b.so
for v in base am4 base am4; do [ $v = base ] && cp /tmp/b.so paper_2512_24449_b200/libpackkv_b200.so || cp tools/exp/lib$v.so paper_2512_24449_b200/libpackkv_b200.so
timeout 600 python bench.py --config C --stream-steps 2048 > /tmp/c.log 2>&1; tail -1 /tmp/c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v C tok/s', d['tokens_per_s'], 'e2e', d['e2e']['tokens_per_s'])"; done
cp /tmp/b.so paper_2512_24449_b200/libpackkv_b200.so
bash tools/exp/ab.sh "s" B base am4 2>&1 | grep -v "^=="
