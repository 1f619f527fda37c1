"""Tree-construction steps of jz-tree written out plainly -- TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2 in the paper's order and notation, with the integer Morton
key reading of DESIGN.md (R4: 21 bits per axis, x most significant, the
paper's float comparator P:L96-101 replaced by integer keys as BASELINE.json
asks). Slow, obviously-correct loops; no blocking or reordering.

  morton_keys      P:L69 (interleave bits), P:L101 (first dimension most significant)
  pair_levels      P:L141-145  lvl_i = lvl(x_{i-1}, x_i), sentinels at i=0 and i=N
  node_ranges      P:L147-155  l_b / r_b by the two searches, n = r_b - l_b
  tree_plane       P:L221-222  splits with n > N_max (boundaries always kept)
  coarser_plane    P:L224      same rule applied to the splits of the previous plane
  plane_schedule   P:L235-243  N_max^(p) = N_max^(0) c^p, stop by N/(N_max/2) < N_target
  dense_ilist      P:L300-305  ispl_i = N i, isrc_j = j mod N
  super_splits     P:L315      Range(0, N_top, NGR)
  radius_of_count  P:L380      smallest radius with cumulative count >= k, else inf
  countheap_insert P:L380      ordered insert, drop last, or merge count (see below)
  node_level       P:L120-124  Morton level of a node: bitlen(first key xor last key); volume 2^lvl
  v90              P:L264-266  point-weighted mean volume of the smallest nodes holding 90% of points
  level_max        P:L260-263  V_max = 2^lvl_max = f_max V_90%: the largest lvl with 2^lvl <= f_max V_90%
  build_hierarchy_reg P:L257-263 regularisation: also split every gap whose level exceeds lvl_max^(p)
"""
from __future__ import annotations

import numpy as np

BITS = 21  # bits per axis (R4)
SENTINEL = 64  # level of the two boundary gaps (> any 63-bit key level; R5)


def key_frame(pos, box=None):
    """Morton frame (R4): periodic -> origin 0, extent L_d per axis; open -> origin =
    FP32 bbox minimum, extent = the largest FP32 span (cubic cells), 1 if all points coincide.
    Returns (origin f32[3], scale f32[3]) with scale_d = RN32(2^21 / extent_d)."""
    pos = np.asarray(pos, dtype=np.float32)
    if box is not None:
        L = np.broadcast_to(np.asarray(box, dtype=np.float64), (3,))
        return np.zeros(3, np.float32), np.array([2.0 ** BITS / l for l in L], dtype=np.float32)
    lo, hi = pos.min(axis=0), pos.max(axis=0)
    e = np.float32(max(np.float32(hi[d] - lo[d]) for d in range(3)))
    if not e > 0:
        e = np.float32(1.0)
    return lo.astype(np.float32), np.full(3, np.float32(2.0 ** BITS / float(e)), dtype=np.float32)


def quantize(pos, origin, scale_or_extent, is_scale=False):
    """q_d = min(trunc(max(RN32(RN32(x_d - o_d) * s_d), 0)), 2^21 - 1), all in FP32
    (R4). Structure only: results never depend on it. With is_scale=False the
    third argument is the extent E and s = RN32(2^21 / E)."""
    pos = np.asarray(pos, dtype=np.float32)
    o = np.broadcast_to(np.asarray(origin, dtype=np.float32), (3,))
    if is_scale:
        s = np.broadcast_to(np.asarray(scale_or_extent, dtype=np.float32), (3,))
    else:
        e = np.broadcast_to(np.asarray(scale_or_extent, dtype=np.float64), (3,))
        s = np.array([2.0 ** BITS / v for v in e], dtype=np.float32)
    v = (pos - o).astype(np.float32) * s
    v = np.clip(v.astype(np.float32), np.float32(0.0), np.float32(2 ** BITS - 1))
    return np.trunc(v).astype(np.uint64)


def morton_keys(q):
    """Interleave: bit b of axis d goes to key bit 3b + (2 - d) (x most significant)."""
    q = np.asarray(q, dtype=np.uint64)
    key = np.zeros(q.shape[0], dtype=np.uint64)
    for b in range(BITS):
        for d in range(3):
            bit = (q[:, d] >> np.uint64(b)) & np.uint64(1)
            key |= bit << np.uint64(3 * b + (2 - d))
    return key


def bitlen(x: int) -> int:
    return int(x).bit_length()


def key_level(a: int, b: int) -> int:
    """Morton level of two keys: number of low bits not shared (P:L120-124 with integer keys)."""
    return bitlen(int(a) ^ int(b))


def pair_levels(keys):
    """N+1 gap levels; gap i lies between sorted points i-1 and i."""
    keys = [int(k) for k in keys]
    n = len(keys)
    lvl = [SENTINEL] * (n + 1)
    for i in range(1, n):
        lvl[i] = key_level(keys[i - 1], keys[i])
    return lvl


def node_ranges(keys):
    """n_i = r_b - l_b for every gap i, by the paper's two searches:
    l_b = smallest index with lvl(x_lb, x_i) <= lvl_i ;
    r_b = smallest index with lvl(x_{i-1}, x_rb) > lvl_i (r_b = N if none).
    Boundary gaps 0 and N get n = +inf (always splits)."""
    keys = [int(k) for k in keys]
    n = len(keys)
    lvl = pair_levels(keys)
    out = [np.inf] * (n + 1)
    for i in range(1, n):
        li = lvl[i]
        lb = 0
        while key_level(keys[lb], keys[i]) > li:  # smallest l_b with level <= lvl_i
            lb += 1
        rb = i
        while rb < n and key_level(keys[i - 1], keys[rb]) <= li:
            rb += 1
        out[i] = rb - lb
    return out


def tree_plane(n_of_gap, nmax):
    """Split gaps (point offsets) of the plane with N_max = nmax."""
    return [g for g, n in enumerate(n_of_gap) if n > nmax]


def coarser_plane(prev_splits, n_of_gap, nmax):
    """Plane p+1 from plane p: keep the splits of plane p with n > nmax,
    returned as positions within the previous split array (Fig. 3: spl^(1) = {0,2,4,5})."""
    return [j for j, g in enumerate(prev_splits) if n_of_gap[g] > nmax]


def plane_schedule(n, nmax0=48, c=8, ntarget=1000):
    """[N_max^(0), N_max^(1), ...] : plane p >= 1 is built while N/(N_max^(p)/2) >= N_target
    (R12); the leaf plane always exists."""
    sched = [nmax0]
    p = 1
    while 2.0 * n / (nmax0 * c ** p) >= ntarget:
        sched.append(nmax0 * c ** p)
        p += 1
    return sched


def build_hierarchy(keys, nmax0=48, c=8, ntarget=1000):
    """All planes for sorted keys. Returns (leaf split gaps, [plane p>=1 splits as
    indices into plane p-1's split array], n per gap)."""
    n_of_gap = node_ranges(keys)
    sched = plane_schedule(len(keys), nmax0, c, ntarget)
    spl0 = tree_plane(n_of_gap, sched[0])
    planes = []
    gaps = spl0
    for nm in sched[1:]:
        idx = coarser_plane(gaps, n_of_gap, nm)
        planes.append(idx)
        gaps = [gaps[j] for j in idx]
    return spl0, planes, n_of_gap


def dense_ilist(nnodes):
    """P:L300-305."""
    ispl = [nnodes * i for i in range(nnodes + 1)]
    isrc = [j % nnodes for j in range(nnodes * nnodes)]
    return ispl, isrc


def super_splits(ntop, ngr=32):
    """Alg. 1 line 1: Range(0, N_top, NGR), closed with N_top."""
    s = list(range(0, ntop, ngr))
    s.append(ntop)
    return s


def radius_of_count(heap, k):
    """smallest radius whose cumulative count >= k; inf if the total < k."""
    tot = 0
    for r, cnt in heap:
        tot += cnt
        if tot >= k:
            return r
    return np.inf


def countheap_insert(heap, r, cnt, k, cap=8):
    """insert keeping radius order and discarding the last element; if discarding
    it would leave a total count < k, add the count to the first element with a larger
    radius instead. (If no element has a larger radius, R13: the last element
    absorbs the count and takes radius r, which keeps the estimate an upper bound.)"""
    h = list(heap)
    pos = 0
    while pos < len(h) and h[pos][0] <= r:
        pos += 1
    if len(h) < cap:
        h.insert(pos, (r, cnt))
        return h
    total = sum(c for _, c in h)
    if total - h[-1][1] + cnt >= k:
        h.insert(pos, (r, cnt))
        h.pop()
        return h
    if pos < len(h):
        h[pos] = (h[pos][0], h[pos][1] + cnt)
    else:
        h[-1] = (r, h[-1][1] + cnt)
    return h


# ----------------------------------------------------------------------------- regularisation
# PAPER.md §2.4 "Regularization". Readings (R18-R20): the volume of a node
# is 2^lvl with lvl its Morton level in bits (the smallest Morton cell holding its first and last
# key; a single point has level 0); V_90%^(p) is computed over the count-based nodes
# of plane p (before any forced split), taken in order of (volume, index) until their cumulative
# point count reaches 90% of all points (the node that crosses 90% is included); lvl_max^(p) is
# made non-decreasing in p so the planes stay nested; f_max is an integer (paper: ~50).


def node_level(keys, a, b):
    """Morton level of the node of sorted points [a, b) (b > a)."""
    return key_level(keys[a], keys[b - 1])


def v90(levels, counts):
    """P:L264-266 as an exact rational (num, den): sum(n_i 2^lvl_i) / sum(n_i) over the smallest
    nodes (by 2^lvl, ties by index) that together contain 90% of all points."""
    total = sum(int(c) for c in counts)
    num = den = 0
    for i in sorted(range(len(levels)), key=lambda j: (int(levels[j]), j)):
        num += int(counts[i]) << int(levels[i])
        den += int(counts[i])
        if 10 * den >= 9 * total:
            break
    return num, den


def level_max(levels, counts, fmax):
    """the largest integer lvl with 2^lvl <= f_max * V_90% (exact integer arithmetic)."""
    num, den = v90(levels, counts)
    lvl = 0
    while (1 << (lvl + 1)) * den <= int(fmax) * num:
        lvl += 1
    return lvl


def build_hierarchy_reg(keys, nmax0=48, c=8, ntarget=1000, fmax=50):
    """Regularised planes: plane p keeps the gaps with n > N_max^(p) and
    also every gap whose level exceeds lvl_max^(p). Returns (leaf split gaps, [plane p >= 1 splits
    as indices into plane p-1's split array], n per gap, [lvl_max^(p)])."""
    keys = [int(k) for k in keys]
    n = len(keys)
    n_of_gap = node_ranges(keys)
    lvl = pair_levels(keys)
    sched = plane_schedule(n, nmax0, c, ntarget)

    def lvl_max_of(splits):
        lv = [node_level(keys, a, b) for a, b in zip(splits[:-1], splits[1:])]
        ct = [b - a for a, b in zip(splits[:-1], splits[1:])]
        return level_max(lv, ct, fmax)

    lm = lvl_max_of(tree_plane(n_of_gap, sched[0]))
    spl0 = [g for g in range(n + 1) if n_of_gap[g] > sched[0] or lvl[g] > lm]
    lms = [lm]
    planes = []
    gaps = spl0
    for nm in sched[1:]:
        lm = max(lvl_max_of([g for g in gaps if n_of_gap[g] > nm]), lm)
        idx = [j for j, g in enumerate(gaps) if n_of_gap[g] > nm or lvl[g] > lm]
        planes.append(idx)
        gaps = [gaps[j] for j in idx]
        lms.append(lm)
    return spl0, planes, n_of_gap, lms
