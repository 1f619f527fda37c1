timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/variants/run2.sh base v2a v2a_l24 v2a_s
