mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C.csv python bench.py --config C --stream-steps 70 --steps 64 --warmup 3 > gpurun_out/launches_C.log 2>&1
tail -1 gpurun_out/launches_C.log | cut -c1-200
