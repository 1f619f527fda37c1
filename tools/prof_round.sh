# Round evidence: launch list of the bench command (cold-cache, serialised), one full capture of
# the top kernel at full size, the sort passes' DRAM bytes, and the bench line itself. $1 = tag
set -x
timeout 900 python bench.py > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/launches_$1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_leaf$ -s 1 -c 1 -o gpurun_out/leaf_$1 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/leaf_$1.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:onesweep -s 8 -c 8 --log-file gpurun_out/sort_dram_$1.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
