cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in gg1k gg8k; do cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
JZ_SKIP_T1=1 JZ_REPS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dl_$v.csv python tools/dist_phases.py 100000000 8 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dl_$v.csv > gpurun_out/dl_$v.txt; echo $v; grep "select_ghosts\|total" gpurun_out/dl_$v.txt
done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -1
