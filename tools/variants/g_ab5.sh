mkdir -p gpurun_out
bash tools/variants/ab.sh "10000000 100000000" cnt0 cnt1 cnt1stats cnt1lcap192 > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
