"""Multi-GPU path on one B200: R logical ranks (threads, in-process exchange) drive every
per-rank stage kernel (Morton keys, splitter bucketing, packing, query boxes, ghost
selection and packing, ghost-carrying build, z-order query) exactly as under torchrun.
Gathered rows must equal the oracle for every R (rank transparency)."""
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
