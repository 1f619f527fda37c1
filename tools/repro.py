import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2604_05885_b200 as jz
from synth import uniform_points
pos = uniform_points(5000, 21, 1.0)
idx, d2 = jz.knn(torch.from_numpy(pos).cuda(), 16, box=1.0)
torch.cuda.synchronize(); print("ok")
