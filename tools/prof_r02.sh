# Round-2 evidence: launch list of the bench command (cold-cache, serialised), one full capture of
# k_leaf at 10^8 (source attributed), DRAM bytes of the build kernels. $1 = tag
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/launches_$tag.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_leaf$ -s 1 -c 1 -o gpurun_out/leaf_$tag python bench.py --profile --steps 1 --warmup 1 > gpurun_out/leaf_$tag.log 2>&1
ncu -i gpurun_out/leaf_$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/leaf_${tag}_cs.csv 2>&1
python tools/ncu_summary.py gpurun_out/leaf_$tag.ncu-rep > gpurun_out/leaf_${tag}_summary.txt 2>&1
ncu -i gpurun_out/leaf_$tag.ncu-rep --page raw --csv > gpurun_out/leaf_${tag}_raw.csv 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:"k_frame|k_hist32|onesweep32|seg_|k_leaf_flags|k_split_n|k_leaf_boxes|k_node_boxes|k_plane" -c 24 --log-file gpurun_out/build_dram_$tag.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
python tools/sort_dram.py gpurun_out/build_dram_$tag.csv 100000000 > gpurun_out/build_dram_${tag}.txt 2>&1
rm -f gpurun_out/leaf_$tag.ncu-rep.bak
echo done
