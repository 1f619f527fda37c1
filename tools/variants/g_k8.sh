cp paper_2604_05885_b200/libjzknn.so /tmp/lib_orig.so
for v in k8m18 k8m20 k8m24; do cp tools/variants/lib_$v.so paper_2604_05885_b200/libjzknn.so
timeout 900 python bench.py --config C5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/c5_$v.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/c5_$v.json')); print('$v', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['stages_ms'].items()})"
done
cp /tmp/lib_orig.so paper_2604_05885_b200/libjzknn.so
