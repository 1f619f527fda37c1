"""Per-rank GPU phases of the multi-GPU path at the size one rank holds at R = 8 (C4: 1.25e7
points), measured on one B200 with CUDA events: local build, query boxes (walk to the leaf plane),
ghost selection, and the final build + query over local + ghosts (ghosts emulated by the
neighbouring z-range of the same data set)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2604_05885_b200 as jz  # noqa: E402
from paper_2604_05885_b200.dist import GpuBackend  # noqa: E402
from synth import make_config  # noqa: E402

n_all = 100_000_000
R = 8
pos, box, k = make_config("C4", n=n_all)
from oracle import tree as T  # noqa: E402  (keys for the host-side emulated partition only)

o, s = T.key_frame(pos[:10], box)
keys = T.morton_keys(T.quantize(pos, o, s, is_scale=True))
order = np.argsort(keys, kind="stable")
m = n_all // R
loc = order[:m]
gh = order[m:m + int(0.15 * m)]
be = GpuBackend()
g = torch.from_numpy(loc.astype(np.int32)).view(torch.float32)
local = torch.cat([torch.from_numpy(pos[loc]), g[:, None]], 1).cuda()
ghosts = torch.cat([torch.from_numpy(pos[gh]), torch.from_numpy(gh.astype(np.int32)).view(torch.float32)[:, None]], 1).cuda()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for rep in range(3):
    torch.cuda.synchronize()
    e0 = ev()
    ix = be.build(local, m, box)
    e1 = ev()
    qb = be.query_boxes(ix, k, 0)
    e2 = ev()
    allb = torch.cat([qb, qb])
    mask, cnt = be.select_ghosts(ix, allb, 1, 2)
    e3 = ev()
    be.free(ix)
    allpts = torch.cat([local, ghosts])
    ix2 = be.build(allpts, m, box)
    e4 = ev()
    out = be.query_z(ix2, k)
    e5 = ev()
    be.free(ix2)
    torch.cuda.synchronize()
    print(f"rep {rep}: build {e0.elapsed_time(e1):.2f} query_boxes {e1.elapsed_time(e2):.2f} select {e2.elapsed_time(e3):.2f} "
          f"build2 {e3.elapsed_time(e4):.2f} query {e4.elapsed_time(e5):.2f} total {e0.elapsed_time(e5):.2f} ms "
          f"(boxes {qb.shape[0]})", flush=True)
