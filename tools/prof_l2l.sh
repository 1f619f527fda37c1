# ncu --set full of the LeafToLeaf kernel on a 10^7-point C4-distribution run (one launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_leaf$ -c 1 -o gpurun_out/l2l_$1 python bench.py --profile --steps 1 --warmup 0 --n 10000000 > gpurun_out/prof_l2l_$1.log 2>&1
echo rc=$?
