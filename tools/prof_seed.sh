cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz
from synth import make_config
pos, box, k = make_config("C4", n=10000000)
ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=box, params=dict(flags=1 << 12)); ix.query(k); ix.free()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_leaf$ -s 1 -c 1 -o gpurun_out/l2l_seed python /tmp/one.py > gpurun_out/prof_seed.log 2>&1
echo rc=$?
