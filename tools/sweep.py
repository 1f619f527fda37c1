"""Sweep tree parameters on the C4 distribution (timing only)."""
import sys, itertools, json, torch, numpy as np
sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz
from synth import make_config
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
grid = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{"nmax0": m} for m in (16, 24, 32, 48, 64)]
pos, box, k = make_config("C4", n=n)
d = torch.from_numpy(pos).cuda()
idx = torch.empty((n, k), dtype=torch.int32, device='cuda'); d2 = torch.empty((n, k), device='cuda')
jz.set_timing(True)
for prm in grid:
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ix = jz.KnnIndex(d, box=box, params=prm); ix.query(k, out=(idx, d2, None))
        e1.record(); torch.cuda.synchronize()
        t = ix.stage_times(); ix.free(); ts.append((e0.elapsed_time(e1), t))
    ms, t = sorted(ts, key=lambda x: x[0])[1]
    print(json.dumps(prm), f"total {ms:7.1f} ms", {kk: round(t[kk], 1) for kk in ("sort", "tree", "node2node", "leaf2leaf")},
          f"evals/q {t['evals']/n:.0f} ins/q {t['inserts']/n:.1f} planes {t['planes']}", flush=True)
