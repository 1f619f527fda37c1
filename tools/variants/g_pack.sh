timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -1
JZ_SKIP_T1=1 JZ_REPS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dl_pack.csv python tools/dist_phases.py 100000000 8 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dl_pack.csv > gpurun_out/dl_pack.txt; head -25 gpurun_out/dl_pack.txt; tail -1 gpurun_out/dl_pack.txt
