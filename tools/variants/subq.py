import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2604_05885_b200 as jz
from synth import make_config
jz.set_timing(True)
pos, box, k = make_config("C4", n=13_600_000)
ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=box)
sp = ix.sorted_points(); ix.free()
n = sp.shape[0]
rng = np.random.default_rng(0)
for frac, mode in [(1.0, "all"), (0.08, "random"), (0.08, "slab")]:
    if mode == "random":
        sel = np.sort(rng.choice(n, int(frac * n), replace=False))
    elif mode == "slab":
        sel = np.arange(int(frac * n))  # a contiguous z range
    else:
        sel = np.arange(n)
    mask = np.zeros(n, bool); mask[sel] = True
    arr = np.concatenate([sp[mask], sp[~mask]])
    t = torch.from_numpy(arr).cuda()
    for rep in range(2):
        i2 = jz.KnnIndex(t, box=box, n_query=len(sel))
        i2.query(k, order="z")
        st = i2.stage_times(); i2.free()
    print(mode, len(sel), {kk: round(v, 2) for kk, v in st.items() if kk in ("sort", "tree", "node2node", "leaf2leaf")}, "planes", st["planes"])
