bash tools/variants/ab.sh "10000000 100000000" pair0 pair1 pair0 pair1 | grep -v "^$"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_pair.log 2>&1; tail -1 gpurun_out/t_pair.log
