# time library variants on the C3 config (10^7 clustered, k = 32)
cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in "$@"; do
  cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
  timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})"
done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
