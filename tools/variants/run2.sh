# time variants at 10^7 and 10^8 with stage split + diag stats (JZ_DIAG_STATS)
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in "$@"; do
  cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
  for n in 10000000 100000000; do
    JZ_DIAG_STATS=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --n $n $BARGS 2>/tmp/err_$v | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['config']['n_points'], round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['stages_ms'].items()}, 'ev/q %.0f' % d['evals_per_query'])"
    grep JZ_STATS /tmp/err_$v | tail -1
  done
done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
