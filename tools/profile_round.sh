#!/bin/bash
# On the GPU box: launch list + full ncu capture of the fused K/V kernels + traffic summary.
# Outputs land in gpurun_out/ (summarised into profiles/ by tools/summarise_profiles.py here).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --nvtx-include "cublas/" \
    --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fast_kernel -s 4 -c 2 -o gpurun_out/prof_full \
    python bench.py --steps 1 --warmup 3 --no-cublas --no-cpu-baseline > gpurun_out/prof_full.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:fast_kernel -s 4 -c 2 --csv --log-file gpurun_out/traffic.csv \
    python bench.py --steps 1 --warmup 3 --no-cublas --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 2 -c 1 -o gpurun_out/prof_single \
    python tools/exp/kbench.py s --cfg B --reps 2 > gpurun_out/prof_single.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C.csv \
    python bench.py --config C --stream-steps 200 --steps 64 --warmup 3 > /dev/null 2>&1
echo done-fused
# compressor: prefill launch list + one full capture of the warp-per-block kernels
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx \
    --nvtx-include "prefill/" --csv --log-file gpurun_out/comp_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:store_fast -c 2 -o gpurun_out/prof_comp \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done-comp
