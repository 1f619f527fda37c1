bash tools/variants/run2.sh novec vec 2>&1 | grep -v JZ_STATS
timeout 900 ncu --set full --clock-control none -k regex:"onesweep32|k_leaf_flags" -s 3 -c 2 -o gpurun_out/sortpass python bench.py --profile --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/sortpass.ncu-rep > gpurun_out/sortpass_summary.txt
ncu -i gpurun_out/sortpass.ncu-rep --page raw --csv > gpurun_out/sortpass_raw.csv
cat gpurun_out/sortpass_summary.txt | grep -E "Duration|Occupancy|Issue|Registers|Throughput|Block Limit"
