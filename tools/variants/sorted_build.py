import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2604_05885_b200 as jz
from synth import make_config
pos, box, k = make_config("C4", n=13_000_000)
d = torch.from_numpy(pos).cuda()
ix = jz.KnnIndex(d, box=box)
sp = torch.from_numpy(ix.sorted_points()).cuda()
ix.free()
def tb(x, nq, label):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        i2 = jz.KnnIndex(x, box=box, n_query=nq); torch.cuda.synchronize()
        dt = (time.perf_counter() - t) * 1e3; i2.free()
    print(label, round(dt, 2), "ms", flush=True)
tb(sp, sp.shape[0], "sorted xyzg")
perm = torch.randperm(sp.shape[0], device="cuda")
tb(sp[perm].contiguous(), sp.shape[0], "shuffled xyzg")
os.environ["JZ_SORT8"] = "1"
