#!/bin/bash
# Bench lines for configs B, A, D, E, C and the reference arm, the GPU tests and smoke (end-of-session refresh).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_B.log 2>&1
for c in A D E; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py --config C > gpurun_out/bench_C.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
for c in B A C D E ref; do tail -1 gpurun_out/bench_$c.log | cut -c1-160; done
