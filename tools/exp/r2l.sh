timeout 900 python -m pytest -q -x tests/test_gpu_fastpath.py tests/test_gpu_single_pass.py 2>&1 | tail -1
bash tools/exp/ab.sh "k v s" B base prev klut
bash tools/exp/ab.sh "k v s" E base prev
