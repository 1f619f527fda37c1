timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for n in 10000000 100000000; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --n $n | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('new', d['config']['n_points'], round(d['ms_per_step'],1), {k:round(v,2) for k,v in d['stages_ms'].items()})"
  JZ_SORT8=1 timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --n $n | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('old', d['config']['n_points'], round(d['ms_per_step'],1), {k:round(v,2) for k,v in d['stages_ms'].items()})"
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k regex:"k_hist32|onesweep32|seg_|k_frame" --log-file gpurun_out/sort_dram_r2c.csv python bench.py --profile --steps 1 --warmup 0 > /dev/null 2>&1
python tools/sort_dram.py gpurun_out/sort_dram_r2c.csv 100000000
