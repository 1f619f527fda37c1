"""Ad-hoc repro: python tools/repro.py <set> <k>  (runs one parity case; use under compute-sanitizer)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2604_05885_b200 as jz
from synth import uniform_points, clustered_points
name = sys.argv[1] if len(sys.argv) > 1 else "clustered"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pos = clustered_points(8000, 23, 1.0) if name == "clustered" else uniform_points(5000, 21, 1.0)
idx, d2 = jz.knn(torch.from_numpy(pos).cuda(), k, box=1.0)
torch.cuda.synchronize()
from oracle import knn_brute
io, do = knn_brute(pos, k, 1.0)
bad = np.nonzero((idx.cpu().numpy() != io).any(1))[0]
print("rows differing:", bad.size, bad[:5])
