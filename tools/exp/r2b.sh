mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_single_pass.py -q -x > gpurun_out/single.log 2>&1; tail -30 gpurun_out/single.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
