mkdir -p gpurun_out
bash tools/variants/ab.sh "10000000 100000000" base exact exactstats > gpurun_out/ab3.txt 2>&1
cat gpurun_out/ab3.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
