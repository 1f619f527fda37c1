python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "passed|failed|Error|C4:|assert" | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['stages_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['e2e']['input_order']['ms_per_step'], d['cpu_baseline'], d['clocks'])"
