mkdir -p gpurun_out
bash tools/variants/ab.sh "10000000 100000000" nodrop drop nodropstats dropstats > gpurun_out/ab2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t2.log 2>&1; tail -3 gpurun_out/t2.log
cat gpurun_out/ab2.txt
