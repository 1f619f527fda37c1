import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2604_05885_b200 as jz
from synth import make_config
jz.set_timing(True)
pos, box, k = make_config("C4")
d = torch.from_numpy(pos).cuda()
for rep in range(12):
    ix = jz.KnnIndex(d, box=box)
    t = ix.stage_times(); ix.free()
    print(rep, round(t["sort"], 2), round(t["tree"], 2), flush=True)
