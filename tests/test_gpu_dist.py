"""Multi-GPU path on one B200: the library's distributed kNN (jz_knn_build_dist /
jz_knn_query_dist) on R logical ranks (threads, the library's in-process communicator) runs the
same code as under torchrun with NCCL: global frame, sampled splitters, Morton-range exchange,
local walk, query boxes from the local k-th distances, ghost exchange, re-walk of the reached
queries, z-order rows (or input order, F2). Gathered rows must equal the oracle for every R
(rank transparency). The NCCL communicator itself runs at one rank."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import knn_grid  # noqa: E402
from synth import clustered_points, uniform_points  # noqa: E402


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("kind,box,k", [("clustered", 1.0, 16), ("uniform", None, 8), ("clustered", None, 32),
                                        ("clustered", 1.0, 48)])
def test_simulated_ranks_equal_oracle(R, kind, box, k):
    from paper_2604_05885_b200.dist import run_ranks_simulated

    gen = clustered_points if kind == "clustered" else uniform_points
    pos = gen(200_000, 17, 1.0)
    idx, d2, owned = run_ranks_simulated(pos, k, box, R)
    assert len(owned) == R and sum(owned) == len(pos)
    io, do = knn_grid(pos, k, box)
    assert np.array_equal(idx, io)
    assert np.array_equal(d2.view(np.int32), do.view(np.int32))


def test_simulated_octant_and_wrap():
    """Adversarial: all points in one octant (one rank holds the others' neighbours) and a
    periodic set whose neighbours wrap between the first and last Morton ranges."""
    from paper_2604_05885_b200.dist import run_ranks_simulated

    p = (uniform_points(50_000, 18, 1.0) * 0.125).astype(np.float32)
    idx, d2, _ = run_ranks_simulated(p, 16, None, 4)
    io, do = knn_grid(p, 16, None)
    assert np.array_equal(idx, io) and np.array_equal(d2, do)
    q = uniform_points(50_000, 19, 1.0)
    q[:, 0] = np.where(q[:, 0] < 0.5, q[:, 0] * 0.02, 1 - (1 - q[:, 0]) * 0.02).astype(np.float32)  # two slabs at x ~ 0 and x ~ 1
    q[:, 0] = np.where(q[:, 0] >= 1.0, 0.0, q[:, 0]).astype(np.float32)
    idx, d2, _ = run_ranks_simulated(q, 16, 1.0, 8)
    io, do = knn_grid(q, 16, 1.0)
    assert np.array_equal(idx, io) and np.array_equal(d2, do)


@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_simulated_ranks_input_order(R):
    """F2: every logical rank returns its own input slice's rows (reverse all-to-all-v through
    jz_bucket_by_splitters / jz_pack_rows / jz_scatter_rows), concatenated = the oracle."""
    from paper_2604_05885_b200.dist import run_ranks_simulated

    pos = clustered_points(120_000, 23, 1.0)
    idx, d2, owned = run_ranks_simulated(pos, 16, 1.0, R, order="input")
    assert owned == [(len(pos) * (r + 1)) // R - (len(pos) * r) // R for r in range(R)]
    io, do = knn_grid(pos, 16, 1.0)
    assert np.array_equal(idx, io)
    assert np.array_equal(d2.view(np.int32), do.view(np.int32))


def test_scatter_rows_rejects_foreign_rows():
    import torch

    from paper_2604_05885_b200 import _binding as B

    rows = torch.zeros((2, 5), dtype=torch.int32, device="cuda")
    rows[:, 4] = torch.tensor([10, 99], dtype=torch.int32)
    oi = torch.empty((5, 2), dtype=torch.int32, device="cuda")
    od = torch.empty((5, 2), dtype=torch.float32, device="cuda")
    rc = B.lib().jz_scatter_rows(B.dptr(rows), 2, 2, 10, 5, B.dptr(oi), B.dptr(od), None)
    assert rc == B.JZ_EDATA and b"outside" in B.lib().jz_last_error()


def test_nccl_comm_one_rank():
    """The NCCL communicator (jz_comm_unique_id / jz_comm_init, libnccl loaded at run time) at
    one rank: the distributed entry points give the single-GPU rows."""
    import ctypes

    import torch

    from paper_2604_05885_b200 import _binding as B
    from paper_2604_05885_b200.dist import Comm, dist_knn

    uid = (ctypes.c_uint8 * 128)()
    B.check(B.lib().jz_comm_unique_id(uid))
    h = ctypes.c_void_p()
    B.check(B.lib().jz_comm_init(uid, 1, 0, ctypes.byref(h)))
    comm = Comm(h)
    pos = clustered_points(50_000, 31, 1.0)
    for order in ("z", "input"):
        idx, d2, rowg = dist_knn(torch.from_numpy(pos).cuda(), 0, 16, 1.0, comm, order=order)
        io, do = knn_grid(pos, 16, 1.0)
        g = rowg.cpu().numpy()
        assert np.array_equal(idx.cpu().numpy(), io[g]) and np.array_equal(d2.cpu().numpy(), do[g])
    comm.free()


def test_dist_ghost_protocol_counts():
    """Ghosts come from the exact local k-th radii (not the count-heap R_max): on the C4
    distribution at R = 8 every rank receives far fewer ghosts than it holds, and only the
    queries of reached boxes are walked twice; rows stay exact."""
    from paper_2604_05885_b200.dist import run_ranks_simulated

    pos = clustered_points(400_000, 37, 1.0)
    stats = []
    idx, d2, owned = run_ranks_simulated(pos, 16, 1.0, 8, stats=stats)
    io, do = knn_grid(pos, 16, 1.0)
    assert np.array_equal(idx, io) and np.array_equal(d2.view(np.int32), do.view(np.int32))
    for _, s in stats:
        assert s["n_local"] > 0 and s["n_ghost"] < s["n_local"] and s["n_requery"] <= s["n_local"]


def test_dist_fewer_than_k_on_a_rank():
    """A rank holding fewer than k points (tiny input split over 8 ranks) answers every query
    through the ghost re-walk (its query boxes have an unbounded radius)."""
    from paper_2604_05885_b200.dist import run_ranks_simulated

    pos = uniform_points(40, 41, 1.0)
    idx, d2, owned = run_ranks_simulated(pos, 12, 1.0, 8)
    io, do = knn_grid(pos, 12, 1.0)
    assert np.array_equal(idx, io) and np.array_equal(d2, do)


def test_dist_bad_input_fails_on_every_rank():
    """A NaN on one rank: that rank reports JZ_EDATA and the peers are released (no hang)."""
    from paper_2604_05885_b200.dist import run_ranks_simulated

    pos = uniform_points(1000, 43, 1.0)
    pos[700, 1] = np.nan
    with pytest.raises(Exception):
        run_ranks_simulated(pos, 4, 1.0, 4)
