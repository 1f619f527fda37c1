bash tools/variants/ab.sh "1000000 10000000 100000000" flat wc
P="import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], d['config']['n_points'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})"
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in flat wc; do cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so; for c in C1 C2 C3; do echo $v; timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --config $c 2>/dev/null | python -c "$P"; done; done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
