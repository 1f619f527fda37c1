for cfg in C2 C3 C5; do for nm in 80 128; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --nmax0 $nm 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg nmax0=$nm', d['config']['n_points'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})"
done; done
