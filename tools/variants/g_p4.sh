bash tools/variants/ab.sh "10000000 100000000" p0 p4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:"k_hist32|onesweep32|seg_" -c 12 --log-file gpurun_out/sort_p4.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
python tools/sort_dram.py gpurun_out/sort_p4.csv 100000000 2>&1 | head -12
