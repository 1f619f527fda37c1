bash tools/variants/ab.sh "1000000 10000000 100000000" nopersist persist
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
