"""F3 measurement: the multivariate normal workload (synth config N1, P:L453 (3)) with and without
the regularisation: device time per build + query, stage times, evals/query."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz  # noqa: E402
from synth import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "N1"
pos, box, k = make_config(cfg)
n = pos.shape[0]
d = torch.from_numpy(pos).cuda()
idx = torch.empty((n, k), dtype=torch.int32, device='cuda')
d2 = torch.empty((n, k), device='cuda')
jz.set_timing(True)
for fmax in (0, 50, 0, 50):
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ix = jz.KnnIndex(d, box=box, params=dict(reg_fmax=fmax))
        ix.query(k, out=(idx, d2, None))
        e1.record()
        torch.cuda.synchronize()
        t = ix.stage_times()
        ix.free()
        ts.append((e0.elapsed_time(e1), t))
    ms, t = sorted(ts, key=lambda x: x[0])[1]
    print(json.dumps({"config": cfg, "n": n, "k": k, "reg_fmax": fmax, "ms": round(ms, 2), "points_per_s": n / ms * 1e3,
                      "stages_ms": {kk: round(t[kk], 2) for kk in ("sort", "tree", "node2node", "leaf2leaf")},
                      "evals_per_query": t["evals"] / n, "leaves": t["leaves"], "planes": t["planes"]}), flush=True)
