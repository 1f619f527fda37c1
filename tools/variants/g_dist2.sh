timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -2
JZ_SKIP_T1=1 JZ_REPS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dist_launches2.csv python tools/dist_phases.py 100000000 8 > gpurun_out/dist_ncu2.log 2>&1
python tools/launch_summary.py gpurun_out/dist_launches2.csv > gpurun_out/dist_launches2.txt; head -12 gpurun_out/dist_launches2.txt; tail -1 gpurun_out/dist_launches2.txt
JZ_REPS=3 timeout 900 python tools/dist_phases.py 100000000 8 > gpurun_out/dist_phases_r02f.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/dist_phases_r02f.json')); print({k:v for k,v in d.items() if k!='ranks'}); [print(r['rank'], round(r['busy_ms'],1), round(r['ghost_frac'],3)) for r in d['ranks']]"
