timeout 900 python -m pytest -q -x tests/test_gpu_single_pass.py 2>&1 | tail -2
bash tools/exp/ab.sh "s" B base ch1 ch8
bash tools/exp/ab.sh "s" E base ch1 ch8
bash tools/exp/ab.sh "s" D base ch8
