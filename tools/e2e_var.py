"""Call-to-call variance of the end-to-end path at 10^8 C4 (k = 16): the C-ABI host call
(jz_knn_search_host_z) against the same work driven from Python over the device API (pinned H2D,
build, query into device tensors, pinned D2H), and the device-only step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_05885_b200 as jz  # noqa: E402
from synth import make_config  # noqa: E402

pos, box, k = make_config("C4")
n = pos.shape[0]
h_pos = torch.from_numpy(pos).pin_memory()
h_idx = torch.empty((n, k), dtype=torch.int32).pin_memory()
h_d2 = torch.empty((n, k), dtype=torch.float32).pin_memory()
h_rg = torch.empty((n,), dtype=torch.int32).pin_memory()
d_idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
d_d2 = torch.empty((n, k), dtype=torch.float32, device="cuda")


def host_api():
    jz.knn_host_z(h_pos.numpy(), k, box=box, out=(h_idx.numpy(), h_d2.numpy(), h_rg.numpy()))


def device_api(copy=True):
    d = h_pos.cuda(non_blocking=True)
    ix = jz.KnnIndex(d, box=box)
    ix.query(k, out=(d_idx, d_d2, None))
    ix.free()
    if copy:
        h_idx.copy_(d_idx, non_blocking=True)
        h_d2.copy_(d_d2, non_blocking=True)


S = torch.cuda.Stream()


def host_api_stream():
    jz.knn_host_z(h_pos.numpy(), k, box=box, out=(h_idx.numpy(), h_d2.numpy(), h_rg.numpy()), stream=S)


def host_api_input():
    jz.knn_host(h_pos.numpy(), k, box=box, out=(h_idx.numpy(), h_d2.numpy()))


which = sys.argv[1:] or ["host_api_z", "host_api_z_stream", "host_api_input", "device_api+copies", "device_only"]
cases = {"host_api_z": host_api, "host_api_z_stream": host_api_stream, "host_api_input": host_api_input,
         "device_api+copies": device_api, "device_only": lambda: device_api(False)}
for name, f in ((w, cases[w]) for w in which):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(name, ts, flush=True)
