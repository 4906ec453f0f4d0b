timeout 900 python -m pytest -q -x tests/test_gpu_fastpath.py tests/test_gpu_parity.py -k "fused or fast or attention or randomized" 2>&1 | tail -1
bash tools/exp/ab.sh "v a" B base prev base prev 2>&1 | grep -v "^=="
bash tools/exp/ab.sh "v a" E base prev 2>&1 | grep -v "^=="
bash tools/exp/ab.sh "v" D base prev 2>&1 | grep -v "^=="
