# source-attributed ncu capture of k_leaf at 10^7 (C4 distribution); $1 = tag
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_leaf$ -c 1 -o gpurun_out/l2l_$1 python bench.py --profile --steps 1 --warmup 0 --n 10000000 > gpurun_out/prof_l2l_$1.log 2>&1
ncu -i gpurun_out/l2l_$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/l2l_$1_cs.csv 2>&1
ncu -i gpurun_out/l2l_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/l2l_$1_sass.csv 2>&1
