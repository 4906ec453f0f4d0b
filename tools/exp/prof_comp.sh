#!/bin/bash
# Compressor only: prefill launch list (time + DRAM bytes) and one full capture of store_fast_compress_kernel.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx \
    --nvtx-include "prefill/" --csv --log-file gpurun_out/comp_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-cublas > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:store_fast -c 2 -o gpurun_out/prof_comp \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-cublas > /dev/null 2>&1
echo done-comp
