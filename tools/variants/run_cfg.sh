# time library variants on a given config: run_cfg.sh CONFIG N VARIANT...
cfg=$1; n=$2; shift 2
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in base "$@"; do
  if [ "$v" != base ]; then cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so; fi
  timeout 300 python bench.py --config $cfg --n $n --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$cfg', d['config']['n_points'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})"
  cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
done
