"""Pins of the friends-of-friends oracle (§5).

The oracle's labels are the connected components of {i ~ j : canonical d2 <= RN32(r_link^2)}
named by their smallest index. Pinned here by hand-worked chains (including the exact
threshold), the periodic wrap, brute force == grid, an independent FP64 graph library
(scipy cKDTree.query_pairs + connected_components, the paper's kind of validator) and
hand-computed catalogue entries."""
import numpy as np
import pytest

from oracle import fof_b2, fof_catalogue, fof_labels
from synth import clustered_points, lattice_points, uniform_points


def _line(xs):
    p = np.zeros((len(xs), 3), np.float32)
    p[:, 0] = xs
    return p


def test_chain_links_and_breaks():
    """Points 0.9 r apart form one group (friends of friends); 1.1 r apart none."""
    r = 0.1
    assert fof_labels(_line(np.arange(20) * 0.09), r, None, "brute").tolist() == [0] * 20
    assert fof_labels(_line(np.arange(20) * 0.11), r, None, "brute").tolist() == list(range(20))


def test_exact_threshold_links():
    """d2 == RN32(r^2) links (<=): r = 0.5, points 0.5 apart -> d2 = 0.25 = b2; one ulp further
    does not (R21)."""
    assert fof_b2(0.5) == np.float32(0.25)
    assert fof_labels(_line([0.0, 0.5, 1.0]), 0.5, None, "brute").tolist() == [0, 0, 0]
    far = np.nextafter(np.float32(0.5), np.float32(1.0))
    assert fof_labels(_line([0.0, far]), 0.5, None, "brute").tolist() == [0, 1]


def test_periodic_wrap_links():
    p = _line([0.99, 0.5, 0.01])
    assert fof_labels(p, 0.05, 1.0, "brute").tolist() == [0, 1, 0]
    assert fof_labels(p, 0.05, None, "brute").tolist() == [0, 1, 2]


def test_labels_are_component_minima():
    p = uniform_points(1500, 41, 1.0)
    lab = fof_labels(p, 0.06, 1.0, "brute")
    idx = np.arange(len(p))
    assert np.all(lab <= idx) and np.array_equal(lab[lab], lab)
    assert np.array_equal(lab[np.unique(lab)], np.unique(lab))


@pytest.mark.parametrize("kind,box", [("uniform", 1.0), ("uniform", None), ("clustered", 1.0), ("clustered", None),
                                      ("dups", 1.0), ("lattice", 1.0)])
def test_grid_equals_brute(kind, box):
    if kind == "uniform":
        p, r = uniform_points(3000, 42, 1.0), 0.05
    elif kind == "clustered":
        p, r = clustered_points(3000, 43, 1.0), 0.2 * 3000 ** (-1 / 3)
    elif kind == "dups":
        q = uniform_points(400, 44, 1.0)
        p, r = np.concatenate([q, q, q[:50]]), 0.03
    else:
        p, r = lattice_points(10, 0.1), 0.1  # every lattice neighbour exactly at r
    assert np.array_equal(fof_labels(p, r, box, "grid"), fof_labels(p, r, box, "brute"))


def test_grid_equals_brute_across_the_wrap():
    """Pairs linked across the periodic face at linking lengths down to the finest grid cell
    (the canonical wrapped t = RN(q - s) +- L carries an absolute error ~ulp(L)/2, R1):
    the grid's cell width keeps every such pair in neighbouring cells."""
    r = np.random.default_rng(5)
    for rl in (1e-3, 1.2e-3, 3e-3):
        pts = []
        for _ in range(400):
            a = r.random(3)
            a[0] = 1.0 - r.random() * rl
            b = a.copy()
            b[0] = (a[0] + rl * (0.9 + 0.2 * r.random())) % 1.0
            pts += [a, b]
        p = np.asarray(pts, np.float32)
        p = np.where(p >= 1, 0, p).astype(np.float32)
        assert np.array_equal(fof_labels(p, rl, 1.0, "grid"), fof_labels(p, rl, 1.0, "brute"))


@pytest.mark.parametrize("box", [1.0, None])
def test_scipy_connected_components(box):
    """Independent FP64 cross-check: same partition as cKDTree.query_pairs + csgraph (no pair is
    within 1e-5 relative of the linking length, so FP32/FP64 rounding cannot differ)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree

    p = clustered_points(4000, 45, 1.0)
    r = 0.2 * 4000 ** (-1 / 3)
    t = cKDTree(p.astype(np.float64), boxsize=box)
    d = t.sparse_distance_matrix(t, r * 1.0001, output_type="ndarray")
    assert not np.any(np.abs(d["v"] - r) < 1e-5 * r), "choose another seed"
    pairs = t.query_pairs(r, output_type="ndarray")
    g = coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(len(p), len(p)))
    _, comp = connected_components(g, directed=False)
    lab = fof_labels(p, r, box)
    # same partition: label -> component is a bijection
    assert len(np.unique(lab)) == len(np.unique(comp))
    assert len(np.unique(lab * (comp.max() + 1) + comp)) == len(np.unique(lab))


def test_catalogue_hand_examples():
    """Square of side 2 centred on (5, 5, 5): centre of mass (5, 5, 5), inertia radius sqrt(2);
    a periodic pair straddling x = 0: centre x = 0 (wrapped), radius 0.01."""
    sq = np.array([[4, 4, 5], [6, 4, 5], [4, 6, 5], [6, 6, 5]], np.float32)
    lab = fof_labels(sq, 2.5, None, "brute")
    u, c, com, rad = fof_catalogue(sq, lab, None, min_count=2)
    assert u.tolist() == [0] and c.tolist() == [4]
    assert np.allclose(com[0], [5, 5, 5], rtol=0, atol=1e-12) and abs(rad[0] - np.sqrt(2)) < 1e-12
    pr = np.array([[0.99, 0.5, 0.5], [0.01, 0.5, 0.5]], np.float32)
    lab = fof_labels(pr, 0.05, 1.0, "brute")
    u, c, com, rad = fof_catalogue(pr, lab, 1.0, min_count=2)
    assert c.tolist() == [2] and abs(com[0, 0] - 0.0) < 1e-7 and abs(rad[0] - 0.01) < 1e-7
    assert fof_catalogue(pr, lab, 1.0, min_count=3)[0].size == 0
