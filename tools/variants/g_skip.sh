bash tools/variants/ab.sh "10000000 100000000" skip0 skip1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
