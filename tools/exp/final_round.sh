#!/bin/bash
# End-of-round measurement: bench lines for configs A-E, the reference arm and the ncu profile round.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_B.log 2>&1
for c in A D E; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py --config C > gpurun_out/bench_C.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
for c in B A C D E ref; do tail -1 gpurun_out/bench_$c.log | cut -c1-200; done
