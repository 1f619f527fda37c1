bash tools/variants/ab.sh "10000000 100000000" fh0 fh1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_fh.log 2>&1; tail -1 gpurun_out/t_fh.log
