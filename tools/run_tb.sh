# parity tests + a quick bench (no e2e / cpu baseline); $1 = tag
timeout 120 python __graft_entry__.py smoke
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests_$1.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests_$1.log
timeout 500 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_$1.log 2>&1; echo bench rc=$?
python - <<'PY' $1
import json,sys
l=open(f"gpurun_out/bench_{sys.argv[1]}.log").read().strip().splitlines()[-1]
d=json.loads(l); print("value %.3e ms %.1f"%(d["value"],d["ms_per_step"]), {k:round(v,2) for k,v in d["stages_ms"].items()}, "evals/q %.0f"%d["evals_per_query"], "frac %.3f"%d["roofline"]["frac"], "ins/q %.1f"%d["inserts_per_query"], {k:round(v,1) for k,v in d["walk_per_item"].items()})
PY
