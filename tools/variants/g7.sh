JZ_REPS=1 JZ_SKIP_T1=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dist_launches8.csv python tools/dist_phases.py 100000000 8 > /dev/null 2>&1
echo rc=$?
