python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2b_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], {k:round(v,2) for k,v in d['stages_ms'].items()}, d['roofline']['frac'], d['e2e']['ms_per_step'], d['e2e']['input_order']['ms_per_step'], d['cpu_baseline']['value'], d['clocks'])"
