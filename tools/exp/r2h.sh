mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_spec_criteria.py 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
