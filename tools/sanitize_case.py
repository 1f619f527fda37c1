"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): exact kNN (periodic and
open, k = 8 / 16 / 40), separate queries, friends-of-friends, two logical ranks of the
distributed path. Each result is checked against the oracle so a clean sanitizer log is also a
parity run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_05885_b200 as jz  # noqa: E402
from oracle import fof_labels, knn_brute  # noqa: E402
from synth import clustered_points, uniform_points  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
ok = []
if which in ("all", "knn"):
    for pos, box, k in [(uniform_points(4096, 1, 1.0), 1.0, 8), (clustered_points(20000, 3, 1.0), 1.0, 16),
                        (uniform_points(20000, 2, 1.0), None, 16), (clustered_points(6000, 5, 1.0), 1.0, 40)]:
        idx, d2 = jz.knn(torch.from_numpy(pos).cuda(), k, box=box)
        io, do = knn_brute(pos, k, box)
        assert np.array_equal(idx.cpu().numpy(), io) and np.array_equal(d2.cpu().numpy(), do)
        ok.append(f"knn n={len(pos)} k={k} box={box}")
if which in ("all", "xq"):
    src, qry = uniform_points(8000, 7, 1.0), uniform_points(3000, 8, 1.0)
    ix = jz.KnnIndex(torch.from_numpy(src).cuda(), box=1.0, queries=torch.from_numpy(qry).cuda())
    idx, d2 = ix.query(8)
    ix.free()
    io, do = knn_brute(src, 8, 1.0, queries=qry)
    assert np.array_equal(idx.cpu().numpy(), io)
    ok.append("separate queries")
if which in ("all", "fof"):
    pos = clustered_points(20000, 9, 1.0)
    lab, _ = jz.fof(torch.from_numpy(pos).cuda(), 0.01, box=1.0, min_count=2)
    assert np.array_equal(lab.cpu().numpy(), fof_labels(pos, 0.01, 1.0))
    ok.append("fof n=20000")
if which in ("all", "dist"):
    from paper_2604_05885_b200.dist import run_ranks_simulated

    pos = clustered_points(20000, 11, 1.0)
    idx, d2, _ = run_ranks_simulated(pos, 16, 1.0, 2)
    io, do = knn_brute(pos, 16, 1.0)
    assert np.array_equal(idx, io)
    ok.append("dist R=2 (logical ranks)")
print("sanitize cases ok:", "; ".join(ok))
