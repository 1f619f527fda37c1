mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
P="import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], d['config']['n_points'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()}, 'ev/q %.0f' % d['evals_per_query'])"
for nm in 64 80 96 112 128; do echo "nmax0 $nm"; timeout 300 $B --nmax0 $nm 2>/dev/null | python -c "$P"; done
for c in C2 C3; do for nm in 80 112; do echo "$c nmax0 $nm"; timeout 300 $B --config $c --nmax0 $nm 2>/dev/null | python -c "$P"; done; done
bash tools/variants/ab.sh "100000000" logx24 exact
