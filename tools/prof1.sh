set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv python bench.py --profile --steps 1 --warmup 0 > gpurun_out/prof_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf2leaf -c 1 -o gpurun_out/l2l_v1 python bench.py --profile --steps 1 --warmup 0 --n 10000000 > gpurun_out/prof_l2l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_n2n -s 6 -c 3 -o gpurun_out/n2n_v1 python bench.py --profile --steps 1 --warmup 0 --n 10000000 > gpurun_out/prof_n2n.log 2>&1
ls -la gpurun_out
