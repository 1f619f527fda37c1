"""Timing ablation of LeafToLeaf mechanisms (debug flag bits << 8; results are wrong)."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz
from synth import make_config
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
pos, box, k = make_config("C4", n=n)
d = torch.from_numpy(pos).cuda()
jz.set_timing(True)
idx = torch.empty((n, k), dtype=torch.int32, device='cuda'); d2 = torch.empty((n, k), device='cuda')
for name, dbg in [("full", 0), ("no-insert", 1), ("no-lanetest", 2), ("no-prepass", 4), ("no-eval", 8), ("no-eval+no-ins", 9)]:
    ts = []
    for rep in range(3):
        ix = jz.KnnIndex(d, box=box, params=dict(flags=dbg << 8))
        ix.query(k, out=(idx, d2, None))
        t = ix.stage_times(); ix.free()
        ts.append(t["leaf2leaf"])
    print(f"{name:16s} leaf2leaf {np.median(ts):7.2f} ms  evals/q {t['evals']/n:6.1f} ins/q {t['inserts']/n:5.1f}", t["walk"])
