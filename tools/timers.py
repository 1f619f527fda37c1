import sys, torch
sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz
from synth import make_config
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
pos, box, k = make_config("C4", n=n)
d = torch.from_numpy(pos).cuda()
jz.set_timing(True)
for dbg in (0, 16, 16):
    ix = jz.KnnIndex(d, box=box, params=dict(flags=dbg << 8)); ix.query(k); t = ix.stage_times(); ix.free()
    print(dbg, "leaf2leaf ms", round(t["leaf2leaf"], 2), flush=True)
