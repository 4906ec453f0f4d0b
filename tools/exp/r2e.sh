timeout 900 python -m pytest -q -x tests/test_gpu_single_pass.py tests/test_gpu_fastpath.py tests/test_gpu_parity.py 2>&1 | tail -3
bash tools/exp/ab.sh "k s a" B base q3
bash tools/exp/ab.sh "k s a" E base q3
