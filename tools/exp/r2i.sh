mkdir -p gpurun_out
cp paper_2512_24449_b200/libpackkv_b200.so /tmp/base.so; cp tools/exp/libw2pred.so paper_2512_24449_b200/libpackkv_b200.so
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize_workload.py > gpurun_out/sanitize_racecheck_w2pred.log 2>&1; tail -2 gpurun_out/sanitize_racecheck_w2pred.log
cp /tmp/base.so paper_2512_24449_b200/libpackkv_b200.so
timeout 900 python bench.py > gpurun_out/bench_B2.log 2>&1; tail -1 gpurun_out/bench_B2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','kernels','attention','e2e','roofline')})"
