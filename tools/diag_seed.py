import sys, torch
sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz
from synth import make_config
n = int(sys.argv[1]); pos, box, k = make_config("C4", n=n)
d = torch.from_numpy(pos).cuda(); jz.set_timing(True)
for f in (0, 1 << 12):
    ix = jz.KnnIndex(d, box=box, params=dict(flags=f)); ix.query(k); t = ix.stage_times(); ix.free()
    print(f, "leaf2leaf(first run) ms", round(t["leaf2leaf"], 2), "evals/q", round(t["evals"] / n), "ins/q", round(t["inserts"] / n, 1), flush=True)
