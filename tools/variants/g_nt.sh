P="import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], d['config']['n_points'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})"
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
for n in 10000000 100000000; do for nt in 300 100 30 10; do echo "n=$n ntarget=$nt"; timeout 300 $B --n $n --ntarget $nt 2>/dev/null | python -c "$P"; done; done
for nt in 300 30; do echo "C3 ntarget=$nt"; timeout 300 $B --config C3 --ntarget $nt 2>/dev/null | python -c "$P"; echo "C2 ntarget=$nt"; timeout 300 $B --config C2 --ntarget $nt 2>/dev/null | python -c "$P"; done
