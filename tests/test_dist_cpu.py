"""World-size-2/3 gloo tests (CPU) of the distributed-kNN protocol that jz_knn_build_dist /
jz_knn_query_dist run inside the library: sample splitters, Morton-range redistribution, query
boxes from the local k-th distances, ghost exchange with reached-box flags, re-walk of the
reached queries, z-order rows with global ids (tests/dist_model.py restates the protocol over
gloo with the CPU stand-ins of tests/cpu_backend.py). The gathered result must equal the
oracle on the whole set (rank transparency). The library's own
implementation is tested with logical ranks on the GPU (tests/test_gpu_dist.py)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import knn_brute
from synth import clustered_points, uniform_points


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, kind, box, k, out_dir, order="z"):
    import torch.distributed as dist

    from tests.cpu_backend import CpuBackend
    from tests.dist_model import TorchComm, dist_knn_model

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gen = uniform_points if kind == "uniform" else clustered_points
    lo, hi = (n * rank) // world, (n * (rank + 1)) // world
    pos = torch.from_numpy(gen(n, 7, 1.0, start=lo, stop=hi))
    if kind == "octant":  # adversarial: everything in one corner, ranks hold each other's neighbours
        pos = pos * 0.125
    idx, d2, rowg = dist_knn_model(pos, lo, k, box, TorchComm(), CpuBackend(), n_samp=64, seed=3, order=order)
    if order == "input":  # F2: this rank's own input slice, in input order
        assert rowg.tolist() == list(range(lo, hi))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), idx=idx.numpy(), d2=d2.numpy(), rowg=rowg.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind,box", [("uniform", 1.0), ("clustered", 1.0), ("clustered", None), ("octant", None)])
def test_gloo_dist_knn_equals_oracle(world, kind, box):
    n, k = 1500, 8
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), n, kind, box, k, d), nprocs=world, join=True)
        idx = np.full((n, k), -1, np.int32)
        d2 = np.zeros((n, k), np.float32)
        owned = []
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            idx[z["rowg"]] = z["idx"]
            d2[z["rowg"]] = z["d2"]
            owned.append(len(z["rowg"]))
    assert sum(owned) == n and min(owned) > 0
    gen = uniform_points if kind == "uniform" else clustered_points
    pos = gen(n, 7, 1.0)
    if kind == "octant":
        pos = (pos * 0.125).astype(np.float32)
    io, do = knn_brute(pos, k, box)
    assert np.array_equal(idx, io)
    assert np.array_equal(d2.view(np.int32), do.view(np.int32))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_dist_knn_input_order(world):
    """F2: rows routed back to the rank owning their input row (reverse all-to-all-v)."""
    n, k = 1200, 8
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), n, "clustered", 1.0, k, d, "input"), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
    idx = np.concatenate([z["idx"] for z in parts])
    d2 = np.concatenate([z["d2"] for z in parts])
    io, do = knn_brute(clustered_points(n, 7, 1.0), k, 1.0)
    assert np.array_equal(idx, io)
    assert np.array_equal(d2.view(np.int32), do.view(np.int32))


def test_splitters_quantiles():
    from tests.dist_model import splitters_from_samples

    s = torch.arange(100, dtype=torch.int64).flip(0)
    spl = splitters_from_samples(s, 4)
    assert spl.tolist() == [25, 50, 75]
    assert splitters_from_samples(s, 1).numel() == 0
