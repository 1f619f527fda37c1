EXTRA="--ntarget 30" bash tools/variants/ab.sh "1000000 10000000 100000000" pre_rc rc
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do JZ_REPS=4 JZ_SKIP_T1=1 timeout 900 python tools/dist_phases.py 100000000 8 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('dist max busy', round(d['max_busy_ms'],1)); [print(r['rank'], round(r['busy_ms'],1), round(r['ghost_frac'],3), {k:round(v,1) for k,v in r['phase_wall_ms'].items()}) for r in d['ranks']]"; done
