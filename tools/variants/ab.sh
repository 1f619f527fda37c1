#!/bin/bash
# A/B timing of library variants (tools/mkvar.py): copies each .so over the in-tree one and runs
# the bench at the given sizes; prints step ms, stage ms, evaluations per query, walk counters.
# usage: bash tools/variants/ab.sh "10000000 100000000" name1 name2 ...
sizes=$1; shift
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in "$@"; do
  cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
  for n in $sizes; do
    timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --n $n $EXTRA 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', d['config']['n_points'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()}, 'ev/q %.0f' % d['evals_per_query'], {k:round(v,1) for k,v in d.get('walk_per_item',{}).items()}, d['clocks'].get('sm_mhz'))"
  done
done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
