timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 600 python tools/dist_phases.py 100000000 8 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:v for k,v in d.items() if k!='ranks'})
for r in d['ranks']: print(r['rank'], r['local'], round(r['ghost_frac'],3), round(r['requery_frac'],3), round(r['busy_ms'],1), {k: round(v,1) for k,v in r['phase_wall_ms'].items()})"
