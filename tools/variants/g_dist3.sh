JZ_SKIP_T1=1 JZ_REPS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dist_launches3.csv python tools/dist_phases.py 100000000 8 > gpurun_out/dist_ncu3.log 2>&1
python tools/launch_summary.py gpurun_out/dist_launches3.csv > gpurun_out/dist_launches3.txt; head -14 gpurun_out/dist_launches3.txt; tail -1 gpurun_out/dist_launches3.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1g.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_1g.csv > gpurun_out/launches_1g.txt; head -8 gpurun_out/launches_1g.txt; tail -1 gpurun_out/launches_1g.txt
grep -i "rank.*local\|n_local" gpurun_out/dist_ncu3.log | head -3
