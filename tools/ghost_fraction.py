"""Ghost fraction of the multi-GPU path: R logical ranks on one B200 (SimComm), C4 distribution;
prints per rank the local and ghost point counts (query boxes: default walk bound, or the
walk-free JZ_FLAG_QBOX_DIAG bound with --diag)."""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2604_05885_b200.dist import GpuBackend, SimComm, SimWorld, dist_knn  # noqa: E402
from synth import make_config  # noqa: E402

n, R = int(sys.argv[1]), int(sys.argv[2])
diag = "--diag" in sys.argv
pos, box, k = make_config("C4", n=n)
bounds = [(n * i) // R for i in range(R + 1)]
world = SimWorld(R)
out = [None] * R


def work(r):
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        be = GpuBackend(params=dict(flags=8) if diag else None, stream=st)
        p = torch.from_numpy(np.ascontiguousarray(pos[bounds[r]:bounds[r + 1]])).cuda()
        t = {}
        dist_knn(p, bounds[r], k, box, SimComm(world, r), be, timings=t)
        st.synchronize()
        out[r] = (t["n_local"], t["n_ghost"])


ths = [threading.Thread(target=work, args=(r,)) for r in range(R)]
[t.start() for t in ths]
[t.join() for t in ths]
for r, (nl, ng) in enumerate(out):
    print(f"rank {r}: local {nl} ghosts {ng} ({100.0 * ng / max(nl, 1):.1f}%)")
