# time library variants: copies each .so over the in-tree one and runs the bench at 10^7 and 10^8
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in "$@"; do
  cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
  for n in 10000000 100000000; do
    timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --n $n 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['config']['n_points'], round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['stages_ms'].items()}, 'ev/q %.0f ins/q %.1f clk %s' % (d['evals_per_query'], d['inserts_per_query'], d['clocks']), {k:round(v,1) for k,v in d['walk_per_item'].items()})"
  done
done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
