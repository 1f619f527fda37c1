"""PCIe floor of the end-to-end call at 10^8 C4 (k = 16): pinned H2D of the positions, pinned D2H of
rows of the real size (one copy and 16 chunks), and the host API itself, all with CUDA events."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_05885_b200 as jz  # noqa: E402
from synth import make_config  # noqa: E402

pos, box, k = make_config("C4")
n = pos.shape[0]


def ev_time(f, reps=3):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


h_pos = torch.from_numpy(pos).pin_memory()
d_pos = torch.empty_like(h_pos, device="cuda")
print("h2d positions %.1f ms" % ev_time(lambda: d_pos.copy_(h_pos, non_blocking=True)))
h_idx = torch.empty((n, k), dtype=torch.int32).pin_memory()
d_idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
print("d2h idx rows (6.4 GB) one copy %.1f ms" % ev_time(lambda: h_idx.copy_(d_idx, non_blocking=True)))
C = 16


def chunks():
    for c in range(C):
        a, b = n * c // C, n * (c + 1) // C
        h_idx[a:b].copy_(d_idx[a:b], non_blocking=True)


print("d2h idx rows 16 chunks %.1f ms" % ev_time(chunks))
h_d2 = torch.empty((n, k), dtype=torch.float32).pin_memory()
h_rg = torch.empty((n,), dtype=torch.int32).pin_memory()
a, b, c, g = h_pos.numpy(), h_idx.numpy(), h_d2.numpy(), h_rg.numpy()
jz.knn_host_z(a, k, box=box, out=(b, c, g))
for _ in range(int(os.environ.get("E2E_REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    jz.knn_host_z(a, k, box=box, out=(b, c, g))
    torch.cuda.synchronize()
    print("knn_host_z wall %.1f ms" % ((time.perf_counter() - t0) * 1e3))
