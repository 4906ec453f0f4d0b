mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_B.log 2>&1; tail -1 gpurun_out/bench_B.log | cut -c1-400
for c in C E; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-300; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
echo done
