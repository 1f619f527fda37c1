"""Ideal-threshold experiment: time LeafToLeaf with every query's k-th d2 known in advance
(variant library built with -DJZ_SEED_EXP). Prints normal vs seeded leaf2leaf ms."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_05885_b200 as jz  # noqa: E402
from paper_2604_05885_b200 import _binding as B  # noqa: E402
from synth import make_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
nmax0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
prm = {"nmax0": nmax0} if nmax0 else None
pos, box, k = make_config("C4", n=n)
d = torch.from_numpy(pos).cuda()
jz.set_timing(True)
lib = B.lib()
lib.jz_exp_seed.argtypes = [ctypes.c_void_p]
res = {}
for mode in ["normal", "normal", "seeded", "seeded"]:
    ix = jz.KnnIndex(d, box=box, params=prm)
    if mode == "seeded":
        lib.jz_exp_seed(ctypes.c_void_p(seed.data_ptr()))
    idx, d2 = ix.query(k)
    t = ix.stage_times()
    lib.jz_exp_seed(ctypes.c_void_p(0))
    ix.free()
    if mode == "normal":
        seed = d2[:, k - 1].contiguous()
        ref = (idx.clone(), d2.clone())
    else:
        assert torch.equal(idx, ref[0]) and torch.equal(d2, ref[1]), "seeded run changed the rows"
    res[mode] = (round(t["leaf2leaf"], 2), t["evals"] / n)
print(n, nmax0, res)
