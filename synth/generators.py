"""Counter-based synthetic inputs (DESIGN.md §"Input recipe").

Every coordinate is a pure function of (seed, point index, draw number), so any
slice [i0, i1) of a data set can be generated independently (each rank of a
multi-GPU run can draw its own contiguous slice, and the global set is the same
for every rank count).

Workloads (BASELINE.json `configs`):
  * uniform   -- coordinates (splitmix64(...) >> 40) * 2^-24 * L: dyadic-exact
                 FP32 values in [0, L).
  * clustered -- Gaussian-halo mixture mimicking a cosmological snapshot
                 (stand-in for the paper's DISCO-DJ snapshots):
                 a fraction f_h = 0.6 of points belongs to halos whose masses
                 follow dN/dM ~ M^-1.9 on [32, 1e-3 N] (drawn until f_h N is
                 covered), centres uniform in the box, isotropic Gaussian
                 profile with sigma = R_vir / 3, R_vir = (3 M / (4 pi 200 nbar))^(1/3).
                 Each point independently picks "halo h with probability
                 M_h / sum M" (prob. f_h) or "background", so the input order is
                 random and any slice is drawable on its own.  Coordinates are
                 formed in float64, wrapped into [0, L) and rounded to float32
                 (a value that rounds up to L maps to 0).
  * lattice   -- n^3 cubic lattice with spacing h (dyadic), for closed-form pins.
"""
from __future__ import annotations

import math
import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

# stream ids (high bits of the counter) so that different draws never collide
_STREAM_POINT = 1
_STREAM_HALO = 2


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied elementwise to uint64 counters."""
    with np.errstate(over="ignore"):
        z = (np.asarray(x, dtype=np.uint64) + _GOLD)
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def _counter(seed: int, stream: int, idx: np.ndarray, draw: int, ndraw: int) -> np.ndarray:
    # counter = seed | stream | (idx * ndraw + draw); idx < 2^34 supported
    base = (np.uint64(seed & 0xFFFF) << np.uint64(48)) | (np.uint64(stream & 0xF) << np.uint64(44))
    return base ^ (idx.astype(np.uint64) * np.uint64(ndraw) + np.uint64(draw))


def _u24(seed, stream, idx, draw, ndraw):
    """Uniform on [0,1) with 24 bits: exactly representable in float32."""
    h = splitmix64(_counter(seed, stream, idx, draw, ndraw))
    return (h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


def _u53(seed, stream, idx, draw, ndraw):
    """Uniform on (0,1) with 53 bits (never exactly 0)."""
    h = splitmix64(_counter(seed, stream, idx, draw, ndraw))
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def _box3(box):
    if box is None:
        return np.ones(3, dtype=np.float64)
    b = np.broadcast_to(np.asarray(box, dtype=np.float64), (3,)).copy()
    return b


def uniform_points(n: int, seed: int, box=None, start: int = 0, stop: int | None = None) -> np.ndarray:
    """Rows [start, stop) of the uniform data set of size n (float32 [m,3])."""
    stop = n if stop is None else stop
    L = _box3(box)
    out = np.empty((stop - start, 3), dtype=np.float32)

    def work(c0, c1):
        idx = np.arange(c0, c1, dtype=np.uint64)
        for d in range(3):
            u = _u24(seed, _STREAM_POINT, idx, d, 8)
            v = (u * L[d]).astype(np.float32)
            v[v >= np.float32(L[d])] = np.float32(0.0)
            out[c0 - start:c1 - start, d] = v

    _parallel_chunks(work, start, stop)
    return out


class _Halos:
    def __init__(self, n: int, seed: int, box, f_halo=0.6, m_min=32.0, slope=1.9, delta=200.0):
        L = _box3(box)
        vol = float(np.prod(L))
        m_max = max(m_min, 1e-3 * n)
        target = f_halo * n
        masses = []
        total = 0.0
        j = 0
        a = 1.0 - slope
        lo, hi = m_min ** a, m_max ** a
        # draw masses in chunks until the halo fraction is covered
        while total < target:
            ids = np.arange(j, j + 4096, dtype=np.uint64)
            u = _u53(seed, _STREAM_HALO, ids, 0, 4)
            m = (lo + u * (hi - lo)) ** (1.0 / a) if m_max > m_min else np.full(ids.shape, m_min)
            c = np.cumsum(m) + total
            k = int(np.searchsorted(c, target, side="left"))
            if k < len(m):
                masses.append(m[: k + 1])
                total = float(c[k])
                j += k + 1
                break
            masses.append(m)
            total = float(c[-1])
            j += len(m)
        self.mass = np.concatenate(masses) if masses else np.zeros(0)
        nh = len(self.mass)
        ids = np.arange(nh, dtype=np.uint64)
        self.center = np.stack([_u53(seed, _STREAM_HALO, ids, 1 + d, 4) * L[d] for d in range(3)], axis=1)
        nbar = n / vol
        r_vir = (3.0 * self.mass / (4.0 * math.pi * delta * nbar)) ** (1.0 / 3.0)
        self.sigma = r_vir / 3.0
        self.cum = np.cumsum(self.mass) / max(total, 1e-300)
        self.f_halo = f_halo
        self.L = L


def clustered_points(n: int, seed: int, box=None, start: int = 0, stop: int | None = None,
                     f_halo: float = 0.6) -> np.ndarray:
    """Rows [start, stop) of the clustered (Gaussian-halo mixture) set of size n."""
    stop = n if stop is None else stop
    halos = _Halos(n, seed, box, f_halo=f_halo)
    L = halos.L
    out = np.empty((stop - start, 3), dtype=np.float32)

    def work(c0, c1):
        idx = np.arange(c0, c1, dtype=np.uint64)
        sel = _u53(seed, _STREAM_POINT, idx, 0, 8)
        in_halo = sel < halos.f_halo
        pos = np.empty((c1 - c0, 3), dtype=np.float64)
        # background: uniform
        for d in range(3):
            pos[:, d] = _u53(seed, _STREAM_POINT, idx, 1 + d, 8) * L[d]
        if len(halos.mass):
            hi = np.nonzero(in_halo)[0]
            ih = idx[hi]
            hid = np.searchsorted(halos.cum, sel[hi] / halos.f_halo, side="right")
            hid = np.minimum(hid, len(halos.mass) - 1)
            # Box-Muller: two pairs of uniforms -> three normals
            u1 = _u53(seed, _STREAM_POINT, ih, 4, 8)
            u2 = _u53(seed, _STREAM_POINT, ih, 5, 8)
            u3 = _u53(seed, _STREAM_POINT, ih, 6, 8)
            u4 = _u53(seed, _STREAM_POINT, ih, 7, 8)
            r1 = np.sqrt(-2.0 * np.log(u1))
            r2 = np.sqrt(-2.0 * np.log(u3))
            sg = halos.sigma[hid]
            cen = halos.center[hid]
            pos[hi, 0] = cen[:, 0] + sg * (r1 * np.cos(2 * math.pi * u2))
            pos[hi, 1] = cen[:, 1] + sg * (r1 * np.sin(2 * math.pi * u2))
            pos[hi, 2] = cen[:, 2] + sg * (r2 * np.cos(2 * math.pi * u4))
        for d in range(3):
            v = pos[:, d] - np.floor(pos[:, d] / L[d]) * L[d]
            f = v.astype(np.float32)
            f[(f >= np.float32(L[d])) | (f < 0)] = np.float32(0.0)
            out[c0 - start:c1 - start, d] = f

    _parallel_chunks(work, start, stop)
    return out


def _parallel_chunks(fn, start, stop, chunk=1 << 20):
    """Run fn(c0, c1) over [start, stop) in chunks on a thread pool (numpy drops the GIL)."""
    spans = [(c0, min(stop, c0 + chunk)) for c0 in range(start, stop, chunk)]
    if len(spans) <= 1:
        for s in spans:
            fn(*s)
        return
    import os
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(spans), os.cpu_count() or 1)) as ex:
        list(ex.map(lambda s: fn(*s), spans))


# fixed lower-triangular factor of the normal workload's covariance (correlated axes)
_NORMAL_A = np.array([[1.0, 0.0, 0.0], [0.5, 0.8, 0.0], [0.2, -0.3, 0.6]])


def normal_points(n: int, seed: int, box=None, start: int = 0, stop: int | None = None) -> np.ndarray:
    """Rows [start, stop) of the multivariate normal set of size n (PAPER.md L453 scenario (3),
    the outlier-heavy case of the regularisation, L257): x = A z, z ~ N(0, I) by double-precision
    Box-Muller, rounded to float32; open domain (`box` is ignored)."""
    stop = n if stop is None else stop
    out = np.empty((stop - start, 3), dtype=np.float32)

    def work(c0, c1):
        idx = np.arange(c0, c1, dtype=np.uint64)
        z = np.empty((c1 - c0, 3))
        for d in range(3):
            u1 = _u53(seed, _STREAM_POINT, idx, 2 * d, 8)
            u2 = _u53(seed, _STREAM_POINT, idx, 2 * d + 1, 8)
            z[:, d] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
        out[c0 - start:c1 - start] = (z @ _NORMAL_A.T).astype(np.float32)

    _parallel_chunks(work, start, stop)
    return out


def lattice_points(n_side: int, h: float = 1.0 / 16.0, jitter_order: bool = False) -> np.ndarray:
    """n_side^3 cubic lattice with spacing h; index = (ix * n + iy) * n + iz."""
    g = np.arange(n_side, dtype=np.float64) * h
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    p = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1).astype(np.float32)
    return p


# BASELINE.json configs: name -> (N, kind, periodic box, k, seed)
CONFIGS = {
    "C1": dict(n=4096, kind="uniform", box=1.0, k=8, seed=1),
    "C2": dict(n=1_000_000, kind="uniform", box=None, k=16, seed=2),
    "C3": dict(n=10_000_000, kind="clustered", box=1.0, k=32, seed=3),
    "C4": dict(n=100_000_000, kind="clustered", box=1.0, k=16, seed=4),
    "C5": dict(n=1 << 30, kind="uniform", box=1.0, k=8, seed=5),
    # aux (not a BASELINE config): the multivariate normal scenario of P:L453 / regularisation P:L257
    "N1": dict(n=10_000_000, kind="normal", box=None, k=16, seed=6),
}


def make_config(name: str, n: int | None = None, start: int = 0, stop: int | None = None):
    """Return (points float32 [m,3], box or None, k) for a named config.

    `n` overrides the size (same distribution family, used for scaled-down tests).
    """
    c = dict(CONFIGS[name])
    if n is not None:
        c["n"] = n
    gen = {"uniform": uniform_points, "clustered": clustered_points, "normal": normal_points}[c["kind"]]
    pts = gen(c["n"], c["seed"], box=c["box"] if c["box"] is not None else 1.0, start=start, stop=stop)
    return pts, c["box"], c["k"]
