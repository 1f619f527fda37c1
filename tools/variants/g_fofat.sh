cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in fofat0 fofat fofat0 fofat; do cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so; echo $v; timeout 600 python tools/fof_bench.py 100000000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms'],1), d['stages_ms'], d.get('groups_ge_20'), d.get('evals_per_point'))"; done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fof" 2>&1 | tail -1
