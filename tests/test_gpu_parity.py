"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar (BASELINE.json north_star): indices bit-exact (ties -> lower index), squared
distances within 1e-6 relative -- asserted here as bit-exact, which the canonical
FP32 formula makes well posed (R1-R3). Sizes span several sort tiles
(3072 keys) and ragged tails; the full-size C4 config is checked on sampled rows.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import knn_brute, knn_grid  # noqa: E402
from oracle import tree as T  # noqa: E402
from synth import clustered_points, lattice_points, make_config, uniform_points  # noqa: E402


def _jz():
    import paper_2604_05885_b200 as jz

    return jz


def _gpu_knn(pos, k, box, order="input", params=None, queries=None):
    jz = _jz()
    t = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.float32)).cuda()
    q = None if queries is None else torch.from_numpy(np.ascontiguousarray(queries, dtype=np.float32)).cuda()
    ix = jz.KnnIndex(t, box=box, params=params, queries=q)
    out = ix.query(k, order=order)
    res = tuple(o.cpu().numpy() for o in out)
    ix.free()
    return res


def _assert_same(idx_g, d2_g, idx_o, d2_o):
    assert idx_g.shape == idx_o.shape
    bad = np.nonzero((idx_g != idx_o).any(axis=1) | (d2_g.view(np.int32) != d2_o.view(np.int32)).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5]}: gpu {idx_g[bad[0]]} {d2_g[bad[0]]} " \
                          f"oracle {idx_o[bad[0]]} {d2_o[bad[0]]}"


def _assert_rel(d2_g, d2_o, tol=1e-6):
    assert np.all(np.abs(d2_g.astype(np.float64) - d2_o) <= tol * np.abs(d2_o.astype(np.float64)))


# ----------------------------------------------------------------------------------- C1


def test_c1_config_bit_exact():
    """C1: 4096 uniform points, unit periodic box, k = 8 vs the brute-force oracle."""
    pos, box, k = make_config("C1")
    ig, dg = _gpu_knn(pos, k, box)
    io, do = knn_brute(pos, k, box)
    _assert_same(ig, dg, io, do)
    _assert_rel(dg, do)


def _sets():
    yield "uniform", uniform_points(5000, 21, 1.0), 1.0
    yield "uniform-open", uniform_points(5000, 22, 1.0), None
    yield "clustered", clustered_points(8000, 23, 1.0), 1.0
    yield "clustered-open", clustered_points(8000, 24, 1.0), None
    d = uniform_points(700, 25, 1.0)
    yield "duplicates", np.concatenate([d, d, d[:100], d[:100], np.repeat(d[:2], 200, axis=0)]), 1.0
    c = np.zeros((1500, 3), np.float32)
    c[:, 0] = uniform_points(1500, 26, 1.0)[:, 0]
    yield "collinear", c, None
    pl = uniform_points(2000, 27, 1.0)
    pl[:, 2] = 0.25
    yield "planar", pl, 1.0
    yield "lattice-periodic", lattice_points(16, 1.0 / 16), 1.0
    yield "lattice-open", lattice_points(12, 0.125), None
    yield "box-faces", np.array([[0, 0, 0], [0.5, 0.5, 0.5], [0.999, 0, 0], [0, 0.999, 0.999], [0.5, 0, 0.999]] * 20,
                                np.float32), 1.0
    yield "anisotropic-box", (uniform_points(3000, 28, 1.0) * np.array([2.0, 1.0, 0.5], np.float32)), (2.0, 1.0, 0.5)
    yield "negative-open", (uniform_points(3000, 29, 1.0) * 8 - 5).astype(np.float32), None
    yield "all-identical", np.full((300, 3), 0.375, np.float32), 1.0


@pytest.mark.parametrize("name,pos,box", list(_sets()), ids=[s[0] for s in _sets()])
@pytest.mark.parametrize("k", [1, 8, 16, 32])
def test_parity_sets(name, pos, box, k):
    if k > len(pos):
        pytest.skip("k > n")
    ig, dg = _gpu_knn(pos, k, box)
    io, do = knn_grid(pos, k, box)
    _assert_same(ig, dg, io, do)


@pytest.mark.parametrize("n", [1, 2, 3, 17, 33, 100, 3071, 3072, 3073, 9217, 65537])
@pytest.mark.parametrize("box", [None, 1.0])
def test_parity_sizes(n, box):
    """Ragged sizes around the radix-sort tile (3072) and warp widths."""
    pos = clustered_points(n, 100 + n, 1.0) if n > 1000 else uniform_points(n, 100 + n, 1.0)
    for k in sorted({1, min(n, 5), min(n, 16), min(n, 32)}):
        ig, dg = _gpu_knn(pos, k, box)
        io, do = knn_grid(pos, k, box)
        _assert_same(ig, dg, io, do)


@pytest.mark.parametrize("params", [dict(nmax0=1), dict(nmax0=8, coarsen=2, ntarget=4), dict(nmax0=32),
                                    dict(nmax0=64, coarsen=3, ntarget=10), dict(nmax0=128), dict(ngr=1),
                                    dict(nmax0=16, coarsen=2, ntarget=1, ngr=3)])
def test_parity_params(params):
    """Tree shape parameters change the walk, never the result."""
    pos = clustered_points(20000, 7, 1.0)
    for box in (1.0, None):
        ig, dg = _gpu_knn(pos, 16, box, params=params)
        io, do = knn_grid(pos, 16, box)
        _assert_same(ig, dg, io, do)


def test_pruning_safety():
    """Disabling the r_low early exit and the segment sort changes no output bit."""
    jz = _jz()
    pos = clustered_points(30000, 8, 1.0)
    ref = _gpu_knn(pos, 16, 1.0)
    for flags in (jz.JZ_FLAG_NO_EARLY_EXIT, jz.JZ_FLAG_NO_SEGSORT, jz.JZ_FLAG_NO_EARLY_EXIT | jz.JZ_FLAG_NO_SEGSORT):
        got = _gpu_knn(pos, 16, 1.0, params=dict(flags=flags))
        assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1].view(np.int32), got[1].view(np.int32))


def test_z_order_rows():
    pos = uniform_points(20000, 9, 1.0)
    ii, di = _gpu_knn(pos, 8, 1.0)
    iz, dz, gz = _gpu_knn(pos, 8, 1.0, order="z")
    assert sorted(gz.tolist()) == list(range(20000))
    assert np.array_equal(iz, ii[gz]) and np.array_equal(dz, di[gz])
    # z order: Morton keys of the rows are non-decreasing
    o, s = T.key_frame(pos, 1.0)
    keys = T.morton_keys(T.quantize(pos[gz], o, s, is_scale=True))
    assert np.all(np.diff(keys.astype(np.float64)) >= 0) or np.all(keys[1:] >= keys[:-1])


def test_query_reuse_and_determinism():
    jz = _jz()
    pos = clustered_points(50000, 10, 1.0)
    t = torch.from_numpy(pos).cuda()
    ix = jz.KnnIndex(t, box=1.0)
    a = [tuple(x.cpu().numpy() for x in ix.query(k)) for k in (16, 8, 16, 32)]
    assert np.array_equal(a[0][0], a[2][0]) and np.array_equal(a[0][1], a[2][1])
    # prefix property across k
    assert np.array_equal(a[1][0], a[0][0][:, :8]) and np.array_equal(a[0][0], a[3][0][:, :16])
    ix.free()


def test_host_entry_point():
    jz = _jz()
    pos = clustered_points(30000, 11, 1.0)
    ih, dh = jz.knn_host(pos, 16, box=1.0)
    ig, dg = _gpu_knn(pos, 16, 1.0)
    assert np.array_equal(ih, ig) and np.array_equal(dh, dg)


def test_errors():
    jz = _jz()
    good = torch.from_numpy(uniform_points(100, 12, 1.0)).cuda()
    with pytest.raises(jz.JzError) as e:
        jz.knn(good, 101, box=1.0)
    assert e.value.code == 2
    with pytest.raises(jz.JzError) as e:
        jz.knn(good[:5], 6, box=1.0)
    assert e.value.code == 2
    bad = good.clone()
    bad[7, 1] = float("nan")
    with pytest.raises(jz.JzError) as e:
        jz.knn(bad, 4)
    assert e.value.code == 3
    out = good.clone()
    out[3, 0] = 1.0  # periodic coordinate must be < L
    with pytest.raises(jz.JzError) as e:
        jz.knn(out, 4, box=1.0)
    assert e.value.code == 3
    with pytest.raises(jz.JzError) as e:
        jz.knn(good, 4, box=(1.0, -1.0, 1.0))
    assert e.value.code == 2
    assert jz.knn(out, 4)[0].shape == (100, 4)  # fine without a box


# ----------------------------------------------------------------------------------- stages


def test_stage_keys_and_sort():
    """A2/A3: GPU keys equal the oracle's Morton keys (same FP32 quantisation, R4)
    and the order is the stable sort of (key, input index)."""
    jz = _jz()
    for box in (1.0, None):
        pos = clustered_points(40000, 13, 1.0)
        if box is None:
            pos = (pos * 3 - 1).astype(np.float32)
        ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=box)
        o, s = T.key_frame(pos, box)
        want = T.morton_keys(T.quantize(pos, o, s, is_scale=True))
        order = np.argsort(want, kind="stable")
        assert np.array_equal(ix.perm(), order)
        assert np.array_equal(ix.sorted_keys(), want[order])
        sp = ix.sorted_points()
        assert np.array_equal(sp[:, :3], pos[order])
        assert np.array_equal(sp[:, 3].view(np.int32), order.astype(np.int32))
        ix.free()


@pytest.mark.parametrize("case", ["short_runs", "cta_runs", "fallback", "near_ties"])
def test_sort_fixup_paths(case):
    """A3 fix-up (DESIGN.md sort): points agreeing in key bits 23..62 are ordered by (key, index)
    by the run fix-up -- in place (runs <= 32), by one CTA (runs <= 2048), or by the 8-pass
    full-key sort (longer runs). Every path must give the stable argsort of the full keys."""
    jz = _jz()
    rng = np.random.default_rng(77)
    base = uniform_points(3000, 21, 1.0)
    if case == "short_runs":  # many runs of 2-6 points inside one 2^-13 cell, distinct low bits
        c = base[rng.integers(0, 3000, 4000)]
        jit = rng.integers(0, 64, (4000, 3)).astype(np.float32) * np.float32(2.0 ** -21)
        pos = np.concatenate([base, (c + jit) % np.float32(1.0)]).astype(np.float32)
    elif case == "cta_runs":  # runs of 40-1500 points in single cells
        parts = [base]
        for m in (40, 300, 1500):
            c = base[rng.integers(0, 3000)]
            jit = rng.integers(0, 256, (m, 3)).astype(np.float32) * np.float32(2.0 ** -21)
            parts.append(((c + jit) % np.float32(1.0)).astype(np.float32))
        pos = np.concatenate(parts)
    elif case == "fallback":  # a run of 3000 identical points: the 8-pass sort
        pos = np.concatenate([base, np.repeat(base[:1], 3000, axis=0)])
    else:  # keys differing only below bit 23 next to exact duplicates
        c = np.repeat(base[:50], 8, axis=0)
        jit = (np.arange(400) % 8)[:, None].astype(np.float32) * np.float32(2.0 ** -21)
        pos = np.concatenate([base, (c + jit) % np.float32(1.0), c]).astype(np.float32)
    pos = rng.permutation(pos).astype(np.float32)
    ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=1.0)
    o, s = T.key_frame(pos, 1.0)
    want = T.morton_keys(T.quantize(pos, o, s, is_scale=True))
    order = np.argsort(want, kind="stable")
    assert np.array_equal(ix.perm(), order)
    assert np.array_equal(ix.sorted_keys(), want[order])
    sp = ix.sorted_points()
    assert np.array_equal(sp[:, :3], pos[order])
    assert np.array_equal(sp[:, 3].view(np.int32), order.astype(np.int32))
    idx, d2 = ix.query(8)
    io, do = knn_brute(pos, 8, 1.0)
    assert np.array_equal(idx.cpu().numpy(), io) and np.array_equal(d2.cpu().numpy().view(np.int32), do.view(np.int32))
    ix.free()


@pytest.mark.parametrize("kind", ["uniform", "clustered", "dups"])
def test_stage_planes_vs_oracle_tree(kind):
    """A4-A7: leaf splits and every coarser plane equal the oracle's hierarchy built by the
    paper's definitions (binary searches, n > N_max^(p)) on the same sorted keys."""
    jz = _jz()
    if kind == "uniform":
        pos = uniform_points(2500, 14, 1.0)
    elif kind == "clustered":
        pos = clustered_points(2500, 15, 1.0)
    else:
        p = uniform_points(500, 16, 1.0)
        pos = np.concatenate([p, p, p[:60], np.repeat(p[:1], 90, axis=0)])
    prm = dict(nmax0=8, coarsen=3, ntarget=20)
    ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=1.0, params=prm)
    keys = ix.sorted_keys()
    spl0, planes, _ = T.build_hierarchy(keys, nmax0=8, c=3, ntarget=20)
    assert ix.num_planes() == 1 + len(planes)
    assert ix.plane_beg(0).tolist() == spl0
    for p, want in enumerate(planes, start=1):
        assert ix.plane_beg(p).tolist() == want
    # A8: boxes are the exact AABBs of the node's points, counts match
    sp = ix.sorted_points()
    beg = ix.plane_beg(0)
    bx = ix.plane_boxes(0)
    for i in range(len(beg) - 1):
        pts = sp[beg[i]:beg[i + 1], :3]
        assert np.array_equal(bx[i, :3], pts.min(axis=0)) and np.array_equal(bx[i, 4:7], pts.max(axis=0))
        assert bx[i, 3:4].view(np.int32)[0] == beg[i + 1] - beg[i]
    ix.free()


@pytest.mark.parametrize("kind,fmax", [("normal", 50), ("normal", 4), ("clustered", 2), ("uniform", 50)])
def test_stage_regularised_planes_vs_oracle(kind, fmax):
    """F3: with reg_fmax the GPU planes equal the oracle's regularised hierarchy
    (lvl_max^(p) from V_90%^(p), forced splits above it) on the same sorted keys; small f_max
    forces many splits, f_max = 50 on uniform points none."""
    from synth import normal_points

    jz = _jz()
    gen = {"normal": normal_points, "clustered": clustered_points, "uniform": uniform_points}[kind]
    pos = gen(3000, 31, 1.0)
    box = 1.0 if kind != "normal" else None
    prm = dict(nmax0=16, coarsen=3, ntarget=20, reg_fmax=fmax)
    ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=box, params=prm)
    keys = ix.sorted_keys()
    spl0, planes, _, _ = T.build_hierarchy_reg(keys, nmax0=16, c=3, ntarget=20, fmax=fmax)
    assert ix.num_planes() == 1 + len(planes)
    assert ix.plane_beg(0).tolist() == spl0
    for p, want in enumerate(planes, start=1):
        assert ix.plane_beg(p).tolist() == want
    ix.free()


@pytest.mark.parametrize("fmax", [50, 2])
def test_regularised_knn_bit_exact(fmax):
    """F3: regularisation changes the tree, never the result (multivariate normal, P:L453 (3))."""
    from synth import normal_points

    pos = normal_points(30000, 32)
    ig, dg = _gpu_knn(pos, 16, None, params=dict(reg_fmax=fmax))
    io, do = knn_brute(pos, 16, None)
    _assert_same(ig, dg, io, do)


# ----------------------------------------------------------------------------------- larger configs


def test_c2_config_full():
    """C2: 10^6 uniform, open boundary, k = 16: every row vs the grid oracle."""
    pos, box, k = make_config("C2")
    ig, dg = _gpu_knn(pos, k, box)
    io, do = knn_grid(pos, k, box)
    _assert_same(ig, dg, io, do)


def test_c3_config_sampled():
    """C3: 10^7 clustered, periodic, k = 32: 20000 sampled rows vs the oracle, invariants on all."""
    pos, box, k = make_config("C3")
    ig, dg = _gpu_knn(pos, k, box)
    rows = np.random.default_rng(3).choice(len(pos), 20000, replace=False)
    io, do = knn_grid(pos, k, box, rows=rows)
    _assert_same(ig[rows], dg[rows], io, do)
    _check_invariants(ig, dg)


def _check_invariants(idx, d2):
    n = idx.shape[0]
    assert np.all(idx >= 0) and np.all(idx < n)
    assert np.all(d2[:, 1:] >= d2[:, :-1])
    tie = d2[:, 1:] == d2[:, :-1]
    assert np.all(idx[:, 1:][tie] > idx[:, :-1][tie])
    assert np.all(d2[:, 0] == 0)


def test_c4_full_size_sampled():
    """C4 at its full size (10^8 clustered, periodic, k = 16) in the bench's launch
    configuration, element by element vs the grid oracle on (a) 10^6 random rows, (b) every row
    whose point lies within 0.002 of a periodic face (wrapped neighbours; ~1.2e6 rows) and
    (c) the 10^4 rows with the smallest k-th distance (halo centres: the densest regions); plus
    the row invariants on all 10^8 rows (on device)."""
    import time

    jz = _jz()
    pos, box, k = make_config("C4")
    t = torch.from_numpy(pos).cuda()
    ix = jz.KnnIndex(t, box=box)
    idx, d2 = ix.query(k)
    ix.free()
    rnd = np.random.default_rng(4).choice(len(pos), 1_000_000, replace=False)
    face = np.nonzero(((pos < 0.002) | (pos > 1 - 0.002)).any(1))[0]
    dense = torch.topk(d2[:, k - 1], 10_000, largest=False).indices.cpu().numpy()  # row choice only
    rows = np.unique(np.concatenate([rnd, face, dense]))
    assert len(face) > 500_000 and len(rows) > 2_000_000
    t0 = time.time()
    io, do = knn_grid(pos, k, box, rows=rows)
    sel = torch.from_numpy(rows).cuda()
    _assert_same(idx[sel].cpu().numpy(), d2[sel].cpu().numpy(), io, do)
    print(f"C4: {len(rows)} rows checked element by element ({len(face)} face rows), oracle {time.time() - t0:.1f} s")
    # invariants on all 10^8 rows, evaluated on the device
    assert bool((idx >= 0).all()) and bool((idx < len(pos)).all())
    assert bool((d2[:, 1:] >= d2[:, :-1]).all())
    tie = d2[:, 1:] == d2[:, :-1]
    assert bool((idx[:, 1:][tie] > idx[:, :-1][tie]).all())
    assert bool((d2[:, 0] == 0).all())


def test_c5_full_size_sampled():
    """C5 at its full size on one B200 (2^30 uniform points, periodic, k = 8; BASELINE.json config 5
    is the 8-GPU run, one GPU holds it: ~60 GB of index + 8.6 GB of rows): sampled rows vs the grid
    oracle over all 2^30 points, plus the row invariants on every row (on device)."""
    jz = _jz()
    pos, box, k = make_config("C5")
    t = torch.from_numpy(pos).cuda()
    ix = jz.KnnIndex(t, box=box)
    idx, d2 = ix.query(k)
    ix.free()
    del t
    rows = np.random.default_rng(5).choice(len(pos), 100_000, replace=False)
    sel = torch.from_numpy(rows).cuda()
    gi, gd = idx[sel].cpu().numpy(), d2[sel].cpu().numpy()
    assert bool((idx >= 0).all()) and bool((idx < len(pos)).all())
    assert bool((d2[:, 1:] >= d2[:, :-1]).all())
    tie = d2[:, 1:] == d2[:, :-1]
    assert bool((idx[:, 1:][tie] > idx[:, :-1][tie]).all())
    assert bool((d2[:, 0] == 0).all())
    del idx, d2, tie
    io, do = knn_grid(pos, k, box, rows=rows)
    _assert_same(gi, gd, io, do)


# ----------------------------------------------------------------------------------- F1
# separate query points (joint tree over both types)
# and k > k_max = 32 (ceil(k/32) LeafToLeaf passes with the (d2, index) lower bound, L386).


def _q_sets():
    yield "uniform", uniform_points(6000, 201, 1.0), uniform_points(4000, 202, 1.0), 1.0
    yield "clustered-src-uniform-q", clustered_points(20000, 203, 1.0), uniform_points(9000, 204, 1.0), 1.0
    yield "uniform-src-clustered-q", uniform_points(5000, 205, 1.0), clustered_points(30000, 206, 1.0), 1.0
    yield "open-q-outside-hull", clustered_points(12000, 207, 1.0), uniform_points(5000, 208, 1.0) * 3 - 1, None
    yield "few-q", clustered_points(40000, 209, 1.0), uniform_points(7, 210, 1.0), None
    yield "few-src", uniform_points(40, 211, 1.0), clustered_points(20000, 212, 1.0), 1.0
    yield "lattice-ties", lattice_points(16, 1.0 / 16), lattice_points(8, 1.0 / 8) + np.float32(1.0 / 32), 1.0
    yield "anisotropic", (uniform_points(8000, 213, 1.0) * np.array([2.0, 1.0, 0.5], np.float32)), \
        (uniform_points(3000, 214, 1.0) * np.array([2.0, 1.0, 0.5], np.float32)), (2.0, 1.0, 0.5)


@pytest.mark.parametrize("name,src,qry,box", list(_q_sets()), ids=[s[0] for s in _q_sets()])
@pytest.mark.parametrize("k", [1, 8, 16, 32])
def test_separate_queries_parity(name, src, qry, box, k):
    if k > len(src):
        pytest.skip("k > n_src")
    ig, dg = _gpu_knn(src, k, box, queries=qry)
    io, do = knn_grid(src, k, box, queries=qry)
    _assert_same(ig, dg, io, do)


def test_separate_queries_small_brute():
    """Sizes spanning the ragged cases: one query, one source, queries == k sources."""
    for ns, nq, k in [(1, 1, 1), (1, 5, 1), (5, 1, 5), (33, 100, 33), (3073, 129, 16), (100, 3073, 100)]:
        for box in (1.0, None):
            src = uniform_points(ns, 300 + ns, 1.0)
            qry = uniform_points(nq, 400 + nq, 1.0)
            ig, dg = _gpu_knn(src, k, box, queries=qry)
            io, do = knn_brute(src, k, box, queries=qry)
            _assert_same(ig, dg, io, do)


def test_separate_queries_z_order_and_empty():
    jz = _jz()
    src = clustered_points(20000, 215, 1.0)
    qry = uniform_points(7000, 216, 1.0)
    ii, di = _gpu_knn(src, 8, 1.0, queries=qry)
    iz, dz, gz = _gpu_knn(src, 8, 1.0, order="z", queries=qry)
    assert sorted(gz.tolist()) == list(range(7000))  # z rows name the query row
    assert np.array_equal(iz, ii[gz]) and np.array_equal(dz, di[gz])
    t = torch.from_numpy(src).cuda()
    ix = jz.KnnIndex(t, box=1.0, queries=torch.empty((0, 3), device="cuda"))
    idx, d2 = ix.query(8)
    assert idx.shape == (0, 8)
    with pytest.raises(jz.JzError) as e:  # k > number of sources
        jz.knn(t[:10], 11, box=1.0, queries=torch.from_numpy(qry).cuda())
    assert e.value.code == 2


def test_xyzg_point_types():
    """jz_knn_build_xyzg type rule: query iff input position < n_query, source iff gidx >= 0
    (a query-only point has gidx < 0; ghosts are source-only points after n_query)."""
    jz = _jz()
    pos = clustered_points(30000, 217, 1.0)
    nq = 18000
    r = np.random.default_rng(5)
    is_src = np.ones(len(pos), bool)
    is_src[:nq] = r.random(nq) < 0.5  # half of the queries are also sources
    gidx = np.full(len(pos), -1, np.int64)
    gidx[is_src] = np.arange(is_src.sum()) * 3 + 7  # monotone in source order: same tie order
    pts4 = np.concatenate([pos, gidx.astype(np.int32).view(np.float32)[:, None]], axis=1)
    ix = jz.KnnIndex(torch.from_numpy(np.ascontiguousarray(pts4)).cuda(), box=1.0, n_query=nq)
    idx, d2 = ix.query(16)
    _, _, rg = ix.query(16, order="z")
    io, do = knn_grid(pos[is_src], 16, 1.0, queries=pos[:nq])
    _assert_same(idx.cpu().numpy(), d2.cpu().numpy(), gidx[is_src][io].astype(np.int32), do)
    # z rows name the query: its gidx when it is also a source, else its input row
    exp = np.where(is_src[:nq], gidx[:nq], np.arange(nq))
    assert np.array_equal(np.sort(rg.cpu().numpy()), np.sort(exp.astype(np.int32)))


@pytest.mark.parametrize("k", [33, 48, 64, 100, 257])
@pytest.mark.parametrize("box", [1.0, None])
def test_large_k_parity(k, box):
    pos = clustered_points(20000, 218, 1.0)
    ig, dg = _gpu_knn(pos, k, box)
    io, do = knn_grid(pos, k, box)
    _assert_same(ig, dg, io, do)


@pytest.mark.parametrize("k", [40, 96])
def test_large_k_ties_and_separate_queries(k):
    """k > 32 on a lattice (many equal distances: the index offset of the pass boundary
    decides) and with separate queries."""
    pos = lattice_points(16, 1.0 / 16)
    ig, dg = _gpu_knn(pos, k, 1.0)
    io, do = knn_brute(pos, k, 1.0)
    _assert_same(ig, dg, io, do)
    src, qry = clustered_points(30000, 219, 1.0), uniform_points(5000, 220, 1.0)
    ig, dg = _gpu_knn(src, k, 1.0, queries=qry)
    io, do = knn_grid(src, k, 1.0, queries=qry)
    _assert_same(ig, dg, io, do)


def test_separate_queries_full_size_sampled():
    """10^7 clustered sources + 10^7 uniform queries (periodic, k = 16): 20000 sampled rows
    vs the grid oracle, invariants on every row."""
    jz = _jz()
    src, box, k = make_config("C3")
    src = src[:10**7]
    qry = uniform_points(10**7, 221, 1.0)
    ix = jz.KnnIndex(torch.from_numpy(src).cuda(), box=box, queries=torch.from_numpy(qry).cuda())
    idx, d2 = ix.query(16)
    rows = np.random.default_rng(9).choice(10**7, 20000, replace=False)
    io, do = knn_grid(src, 16, box, rows=rows, queries=qry)
    _assert_same(idx[rows].cpu().numpy(), d2[rows].cpu().numpy(), io, do)
    d = d2.double()
    assert bool((d[:, 1:] >= d[:, :-1]).all()) and bool(torch.isfinite(d).all())
    assert int(idx.min()) >= 0 and int(idx.max()) < 10**7


# ----------------------------------------------------------------------------------- F4 friends-of-friends
def _fof_cmp(pos, r, box, min_count=20):
    from oracle import fof_catalogue, fof_labels

    jz = _jz()
    lab, cat = jz.fof(torch.from_numpy(np.ascontiguousarray(pos)).cuda(), r, box=box, min_count=min_count)
    lab = lab.cpu().numpy()
    want = fof_labels(pos, r, box)
    assert np.array_equal(lab, want), f"{(lab != want).sum()} labels differ"
    u, c, com, rad = fof_catalogue(pos, want, box, min_count)
    order = np.argsort(cat["label"].cpu().numpy(), kind="stable")
    assert np.array_equal(cat["label"].cpu().numpy()[order], u)
    assert np.array_equal(cat["count"].cpu().numpy()[order], c)
    got_com = cat["com"].cpu().numpy()[order]
    if box is not None:  # compare on the circle: a centre at ~0 may come back as ~L
        dd = got_com - com
        L = np.broadcast_to(np.asarray(box, np.float64), (3,))
        dd -= L * np.round(dd / L)
        assert np.abs(dd).max(initial=0) <= 1e-9
    else:
        assert np.allclose(got_com, com, rtol=1e-9, atol=1e-12)
    assert np.allclose(cat["rad"].cpu().numpy()[order], rad, rtol=1e-7, atol=1e-12)
    return len(np.unique(want))


@pytest.mark.parametrize("kind,box", [("uniform", 1.0), ("uniform", None), ("clustered", 1.0), ("clustered", None),
                                      ("dups", 1.0), ("lattice", 1.0), ("normal", None)])
def test_fof_labels_and_catalogue(kind, box):
    """F4: labels bit-identical to the oracle's components, catalogue (count exact;
    centre of mass / inertia radius FP64 within 1e-9 / 1e-7 relative: atomics sum in any order)."""
    from synth import normal_points

    if kind == "uniform":
        pos, r = uniform_points(60000, 51, 1.0), 0.2 * 60000 ** (-1 / 3) * 3
    elif kind == "clustered":
        pos, r = clustered_points(80000, 52, 1.0), 0.2 * 80000 ** (-1 / 3)
    elif kind == "dups":
        q = uniform_points(3000, 53, 1.0)
        pos, r = np.concatenate([q, q, q[:500], np.repeat(q[:2], 300, axis=0)]), 0.02
    elif kind == "lattice":
        pos, r = lattice_points(16, 1.0 / 16), 1.0 / 16  # every lattice neighbour exactly at r: one group
    else:
        pos, r = normal_points(50000, 54), 0.05
    ng = _fof_cmp(pos, r, box, min_count=2)
    assert ng >= 1


def test_fof_extremes_and_errors():
    """r = 0 links only exact duplicates; a huge r links everything; FoF on a separate-query index
    is refused."""
    jz = _jz()
    q = uniform_points(2000, 55, 1.0)
    pos = np.concatenate([q, q[:100]])
    _fof_cmp(pos, 0.0, 1.0, min_count=2)
    lab, cat = jz.fof(torch.from_numpy(pos).cuda(), 2.0, box=None, min_count=1)
    assert (lab.cpu().numpy() == 0).all() and cat["count"].cpu().tolist() == [len(pos)]
    ix = jz.KnnIndex(torch.from_numpy(q).cuda(), box=1.0, queries=torch.from_numpy(q[:10]).cuda())
    with pytest.raises(Exception):
        ix.fof(0.01)
    ix.free()


def test_fof_c4_distribution_full():
    """F4 on 10^6 points of the C4 (clustered) distribution, b = 0.2 mean separations, every
    label vs the grid oracle."""
    pos, box, _ = make_config("C4", n=1_000_000)
    _fof_cmp(pos, 0.2 * 1e6 ** (-1 / 3), box, min_count=20)


# ----------------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("n,k,box", [(1, 1, 1.0), (2, 2, None), (3, 1, 1.0), (40, 40, 1.0), (33, 33, None),
                                     (100, 64, 1.0), (257, 8, None)])
def test_tiny_and_k_equals_n(n, k, box):
    """Degenerate sizes: one point, k = n (every point in every row, including k > 32 = k_max
    passes), a ragged tail of the 32-query work items."""
    pos = uniform_points(n, 300 + n, 1.0)
    ig, dg = _gpu_knn(pos, k, box)
    io, do = knn_brute(pos, k, box)
    _assert_same(ig, dg, io, do)


@pytest.mark.parametrize("offset,scale", [(1.0e6, 1.0), (-3.0e5, 50.0), (1.0e-3, 1.0e-6)])
def test_far_offsets_and_tiny_scales(offset, scale):
    """Open domain far from the origin (coordinates ~1e6 with unit spread: FP32 spacing ~0.06) and
    a microscopic cloud: the rounding margins of the pruning bounds (R8b) must keep every
    true neighbour."""
    pos = (uniform_points(20000, 310, 1.0).astype(np.float64) * scale + offset).astype(np.float32)
    ig, dg = _gpu_knn(pos, 16, None)
    io, do = knn_brute(pos, 16, None)
    _assert_same(ig, dg, io, do)


def test_periodic_points_near_the_box_faces():
    """Periodic box with most points within 1e-4 of the faces: every leaf pair straddles or wraps
    (per-pair select and shift classes, R8b)."""
    p = uniform_points(30000, 311, 1.0).astype(np.float64)
    p = np.where(p < 0.5, p * 2e-4, 1.0 - (1.0 - p) * 2e-4).astype(np.float32)
    p[p >= np.float32(1.0)] = np.float32(0.0)  # float32 rounding can reach L
    ig, dg = _gpu_knn(p, 16, 1.0)
    io, do = knn_grid(p, 16, 1.0)
    _assert_same(ig, dg, io, do)


def test_search_host_z_streamed():
    """jz_knn_search_host_z: rows in z order streamed to host memory in chunks during the walk;
    row r answers input point row_gidx[r] exactly as the oracle (and as the input-order call)."""
    import paper_2604_05885_b200 as jz

    for pos, box, k in [(uniform_points(300_000, 51, 1.0), None, 16), (clustered_points(200_000, 52, 1.0), 1.0, 8),
                        (clustered_points(50_000, 53, 1.0), 1.0, 40)]:
        idx, d2, rg = jz.knn_host_z(pos, k, box=box)
        assert np.array_equal(np.sort(rg), np.arange(len(pos)))
        io, do = knn_grid(pos, k, box)
        _assert_same(idx, d2, io[rg], do[rg])


@pytest.mark.parametrize("kind,box,r", [("clustered", 1.0, 0.01), ("uniform", None, 0.02), ("clustered", 1.0, 0.3)])
def test_fof_group_order(kind, box, r):
    """P:L498 group order: a stable sort of the points by group root -- every group (oracle
    components) is one contiguous block, blocks in z order of their roots, z order inside."""
    import paper_2604_05885_b200 as jz
    from oracle import fof_labels

    pos = (clustered_points if kind == "clustered" else uniform_points)(30_000, 61, 1.0)
    ix = jz.KnnIndex(torch.from_numpy(pos).cuda(), box=box)
    lab, _ = ix.fof(r, 2)
    order, beg = ix.fof_group_order()
    perm = ix.perm()
    ix.free()
    order, beg, lab = order.cpu().numpy(), beg.cpu().numpy(), lab.cpu().numpy()
    want = fof_labels(pos, r, box)
    assert np.array_equal(lab, want)
    assert np.array_equal(np.sort(order), np.arange(len(pos)))
    zpos = np.empty(len(pos), np.int64)
    zpos[perm] = np.arange(len(pos))
    assert beg[0] == 0 and beg[-1] == len(pos) and np.all(np.diff(beg) > 0)
    assert len(beg) - 1 == len(np.unique(want))
    heads = []
    for g in range(len(beg) - 1):
        blk = order[beg[g]:beg[g + 1]]
        assert np.all(want[blk] == want[blk[0]])
        assert np.all(np.diff(zpos[blk]) > 0)
        heads.append(zpos[blk[0]])
    assert np.all(np.diff(heads) > 0)
