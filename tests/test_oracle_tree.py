"""Pins for oracle/tree.py (CPU only): the paper's Fig. 3 worked example, SPEC worked
examples, and properties that follow from the definitions (cell containment,
nearest-strictly-greater equivalence, nesting of planes)."""
import math

import numpy as np
import pytest

from oracle import tree as T
from synth import clustered_points, uniform_points


def _fig3_keys(g):
    x = np.array(g["x"], dtype=np.float32)
    pos = np.zeros((len(x), 3), np.float32)
    pos[:, 0] = x / np.float32(16.0)  # exact (power of two)
    keys = T.morton_keys(T.quantize(pos, 0.0, 1.0))
    return keys


def test_fig3_levels(golden):
    """interior lvl = [2,-1,3,1,2,4,0] in the paper's 1-D float convention
    maps to integer-key levels 3*lvl + 51 under the embedding (SURVEY SV-3)."""
    g = golden("fig3.json")
    keys = _fig3_keys(g)
    assert list(keys) == sorted(keys)  # already z-sorted (1-D: numeric order)
    lv = T.pair_levels(keys)
    assert lv[0] == T.SENTINEL and lv[-1] == T.SENTINEL
    assert [l - 51 for l in lv[1:-1]] == [3 * l for l in g["paper_lvl_interior"]]


def test_fig3_node_sizes_and_planes(golden):
    """n = [3,2,6,2,3,8,2]; spl^(0) (n>2) = {0,1,3,5,6,8}; spl^(1) (n>4) = {0,2,4,5}."""
    g = golden("fig3.json")
    keys = _fig3_keys(g)
    n = T.node_ranges(keys)
    assert n[1:-1] == g["n_interior"]
    spl0 = T.tree_plane(n, g["nmax0"])
    assert spl0 == g["spl0"]
    assert T.coarser_plane(spl0, n, g["nmax1"]) == g["spl1"]
    s0, planes, _ = T.build_hierarchy(keys, nmax0=2, c=2, ntarget=1)
    assert s0 == g["spl0"] and planes[0] == g["spl1"]


def test_morton_bit_layout():
    """x most significant: bit b of x -> key bit 3b+2, y -> 3b+1, z -> 3b."""
    q = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [2, 0, 0], [0, 0, 2], [2 ** 21 - 1] * 3], np.uint64)
    assert T.morton_keys(q).tolist() == [4, 2, 1, 32, 8, 2 ** 63 - 1]


def test_morton_grid_z_pattern():
    """Fig. zorder: on a regular 4x4 grid (z = 0) the sorted order visits
    2x2 blocks in a Z, first dimension most significant."""
    g = np.array([[x, y, 0] for x in range(4) for y in range(4)], np.uint64)
    order = np.argsort(T.morton_keys(g), kind="stable")
    got = [tuple(int(v) for v in g[i][:2]) for i in order]
    assert got[:4] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert got[4:8] == [(0, 2), (0, 3), (1, 2), (1, 3)]


def test_quantize_clamps():
    q = T.quantize(np.array([[0.0, 0.5, 0.99999994]], np.float32), 0.0, 1.0)
    assert q.tolist() == [[0, 2 ** 20, 2 ** 21 - 1]]


def _nearest_greater_n(lvl):
    n = len(lvl) - 1
    out = [math.inf] * (n + 1)
    for i in range(1, n):
        L = i - 1
        while lvl[L] <= lvl[i]:
            L -= 1
        R = i + 1
        while lvl[R] <= lvl[i]:
            R += 1
        out[i] = R - L
    return out


@pytest.mark.parametrize("kind", ["uniform", "clustered", "dups"])
def test_node_ranges_equal_nearest_greater(kind):
    """The binary-search definition equals 'distance between the nearest
    strictly greater gap levels' (SURVEY SV-3), and every node is a Morton cell:
    its points share key bits >= lvl."""
    if kind == "uniform":
        pos = uniform_points(300, 3, 1.0)
    elif kind == "clustered":
        pos = clustered_points(300, 4, 1.0)
    else:
        p = uniform_points(60, 5, 1.0)
        pos = np.concatenate([p, p, p[:10], p[:10], p[:10]])
    keys = np.sort(T.morton_keys(T.quantize(pos, 0.0, 1.0)))
    n_bs = T.node_ranges(keys)
    lvl = T.pair_levels(keys)
    assert n_bs == _nearest_greater_n(lvl)
    kl = [int(k) for k in keys]
    for i in range(1, len(kl)):
        # cell of gap i: contiguous run of keys with equal (key >> lvl_i)
        sh = lvl[i]
        members = [j for j in range(len(kl)) if (kl[j] >> sh) == (kl[i] >> sh)]
        assert members == list(range(members[0], members[-1] + 1))
        assert len(members) == n_bs[i]


def test_plane_nesting_and_capacity():
    """Planes nest (each coarse split is a finer split) and every node of plane p holds
    <= N_max^(p) points."""
    pos = clustered_points(3000, 9, 1.0)
    keys = np.sort(T.morton_keys(T.quantize(pos, 0.0, 1.0)))
    spl0, planes, n = T.build_hierarchy(keys, nmax0=8, c=4, ntarget=10)
    assert spl0[0] == 0 and spl0[-1] == len(keys)
    gaps = spl0
    cap = 8
    assert max(np.diff(gaps)) <= cap
    for idx in planes:
        cap *= 4
        assert idx[0] == 0 and idx[-1] == len(gaps) - 1
        gaps = [gaps[j] for j in idx]
        assert max(np.diff(gaps)) <= cap


def test_plane_schedule():
    """P:L235-243 with defaults 48 / 8 / 1000 (plane p >= 1 iff 2N / (48 8^p) >= 1000):
    10^8 points -> 5 planes, 10^7 -> 3, 10^6 -> 2, 4096 -> 1."""
    assert T.plane_schedule(10 ** 8) == [48, 384, 3072, 24576, 196608]
    assert len(T.plane_schedule(10 ** 7)) == 3
    assert T.plane_schedule(10 ** 6) == [48, 384]
    assert T.plane_schedule(4096) == [48]


def test_spec_ilist_and_countheap_examples(golden):
    g = golden("spec_examples.json")
    for n, want in g["dense_init"].items():
        ispl, isrc = T.dense_ilist(int(n))
        assert ispl == want["ispl"] and isrc == want["isrc"]
    for ntop, ngr, want in g["super_splits"]:
        assert T.super_splits(ntop, ngr) == want
    for heap, k, want in g["radius_of_count"]:
        r = T.radius_of_count([tuple(e) for e in heap], k)
        assert (math.isinf(r) and want == "inf") or r == want
    for case in g["countheap_insert"]:
        h = T.countheap_insert([tuple(e) for e in case["heap"]], *case["insert"], k=case["k"], cap=case["cap"])
        assert [list(e) for e in h] == case["out"]


def test_countheap_radius_is_upper_bound():
    """After any sequence of inserts, every radius r' >= RadiusOfCount still covers at
    least as many counted items as the truth: the estimate never undercounts
    (the property FindRmax relies on)."""
    rng = np.random.default_rng(2)
    for trial in range(200):
        k = int(rng.integers(1, 40))
        items = [(float(rng.random()), int(rng.integers(1, 10))) for _ in range(int(rng.integers(1, 30)))]
        h = []
        for r, c in items:
            if r < T.radius_of_count(h, k):
                h = T.countheap_insert(h, r, c, k, cap=8)
        R = T.radius_of_count(h, k)
        true_cnt = sum(c for r, c in items if r <= R)
        if math.isfinite(R):
            assert true_cnt >= k
        else:
            assert sum(c for _, c in items) < k  # every item was inserted; counts are conserved


# ------------------------------------------------------------------ regularisation
def test_reg_v90_hand_examples():
    """P:L260-266 worked by hand: four level-3 nodes of 4 points and a level-20 outlier node of 1:
    the smallest nodes reach 16/17 >= 90% without the outlier, so V_90% = 2^3 = 8 and
    f_max = 50 gives V_max = 400 -> lvl_max = 8 (2^8 = 256 <= 400 < 512)."""
    assert T.v90([3, 3, 3, 3, 20], [4, 4, 4, 4, 1]) == (128, 16)
    assert T.level_max([3, 3, 3, 3, 20], [4, 4, 4, 4, 1], 50) == 8
    assert T.level_max([3, 3, 3, 3, 20], [4, 4, 4, 4, 1], 1) == 3
    # ties in volume are taken in index order; the node crossing 90% is included:
    # total 21, 0.9 * 21 = 18.9 -> nodes (lvl 2, n 1), (lvl 5, n 10), (lvl 5, n 10)
    assert T.v90([5, 2, 5], [10, 1, 10]) == (4 + 320 + 320, 21)
    assert T.level_max([5, 2, 5], [10, 1, 10], 50) == 10  # 50 * 644 / 21 = 1533.3 -> 2^10


def _keys_of(pos, box=None):
    o, s = T.key_frame(pos, box)
    return np.sort(T.morton_keys(T.quantize(pos, o, s, is_scale=True)))


def test_reg_splits_isolate_outliers():
    """a multivariate normal set (P:L453 (3)): count-based leaves in the sparse tails span
    huge Morton cells; the regularised plane splits every gap above lvl_max, so every node of >= 2 points has
    level <= lvl_max (its level is its largest interior gap), it refines the count-based plane,
    and here it has more leaves."""
    from synth import normal_points

    keys = [int(k) for k in _keys_of(normal_points(3000, 6))]
    n_of_gap = T.node_ranges(keys)
    base = T.tree_plane(n_of_gap, 48)
    spl0, planes, _, lms = T.build_hierarchy_reg(keys, nmax0=48, c=8, ntarget=1, fmax=50)
    assert set(base) <= set(spl0) and len(spl0) > len(base)
    for a, b in zip(spl0[:-1], spl0[1:]):
        if b - a >= 2:
            assert T.node_level(keys, a, b) <= lms[0]
    big = max(T.node_level(keys, a, b) for a, b in zip(base[:-1], base[1:]))
    assert big > lms[0]  # without the regularisation some leaf exceeds V_max
    gaps = spl0
    for p, idx in enumerate(planes):  # nested, and the level bound holds on every plane
        sub = [gaps[j] for j in idx]
        assert set(sub) <= set(gaps) and lms[p + 1] >= lms[p]
        for a, b in zip(sub[:-1], sub[1:]):
            if b - a >= 2:
                assert T.node_level(keys, a, b) <= lms[p + 1]
        gaps = sub


def test_reg_uniform_unchanged():
    """for uniform random points the count-based structure is already regular:
    f_max = 50 adds no split."""
    from synth import uniform_points

    keys = [int(k) for k in _keys_of(uniform_points(4000, 9, 1.0), 1.0)]
    spl0, planes, n_of_gap, _ = T.build_hierarchy_reg(keys, nmax0=48, c=8, ntarget=10, fmax=50)
    s0, p0, _ = T.build_hierarchy(keys, nmax0=48, c=8, ntarget=10)
    assert spl0 == s0 and planes == p0
