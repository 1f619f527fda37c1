"""ctypes front end of the C oracle (jz_oracle.c). TEST INFRASTRUCTURE ONLY.

Definition computed (PAPER.md L295/L432/L453-454): for each query
row i the k smallest (d2, j) over all points j (self included, ties -> lower j),
d2 the canonical FP32 formula  fmaf(dz,dz,fmaf(dy,dy,dx*dx)),  dx = RN(q-s)
wrapped to the minimal image [-L/2, L/2) when a periodic box is given.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jz_oracle.c")
_BUILD = os.path.join(_HERE, "_build")
_LIB = os.path.join(_BUILD, "libjzoracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build_oracle(force: bool = False) -> str:
    """Compile jz_oracle.c into oracle/_build/libjzoracle.so (if stale)."""
    os.makedirs(_BUILD, exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_oracle())
            P = ctypes.c_void_p
            lib.oracle_knn_brute.argtypes = [P, ctypes.c_int64, P, ctypes.c_int, P, ctypes.c_int64, P, P, ctypes.c_int]
            lib.oracle_knn_brute.restype = ctypes.c_int
            lib.oracle_knn_grid.argtypes = [P, ctypes.c_int64, P, ctypes.c_int, P, ctypes.c_int64, P, P,
                                            ctypes.c_int, ctypes.c_double]
            lib.oracle_knn_grid.restype = ctypes.c_int
            lib.oracle_knn_brute_q.argtypes = [P, ctypes.c_int64, P, P, ctypes.c_int, P, ctypes.c_int64, P, P,
                                               ctypes.c_int]
            lib.oracle_knn_brute_q.restype = ctypes.c_int
            lib.oracle_knn_grid_q.argtypes = [P, ctypes.c_int64, P, P, ctypes.c_int, P, ctypes.c_int64, P, P,
                                              ctypes.c_int, ctypes.c_double]
            lib.oracle_knn_grid_q.restype = ctypes.c_int
            lib.oracle_pair_d2.argtypes = [P, P, ctypes.c_int64, P, P]
            lib.oracle_pair_d2.restype = None
            lib.oracle_fof_brute.argtypes = [P, ctypes.c_int64, P, ctypes.c_float, P]
            lib.oracle_fof_brute.restype = ctypes.c_int
            lib.oracle_fof_grid.argtypes = [P, ctypes.c_int64, P, ctypes.c_float, P]
            lib.oracle_fof_grid.restype = ctypes.c_int
            lib.oracle_max_threads.argtypes = []
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def oracle_threads() -> int:
    return int(_load().oracle_max_threads())


def _prep(pos, box):
    pos = np.ascontiguousarray(pos, dtype=np.float32)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ValueError("pos must be [n,3]")
    b = None
    if box is not None:
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(box, dtype=np.float32), (3,)))
    return pos, b


def _ptr(a):
    return None if a is None else a.ctypes.data


def _run(fn, pos, k, box, rows, threads, *extra, queries=None):
    pos, b = _prep(pos, box)
    n = pos.shape[0]
    qry = None
    if queries is not None:
        qry, _ = _prep(queries, None)
    if rows is None:
        nrows, r = (n if qry is None else qry.shape[0]), None
    else:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        nrows = r.shape[0]
    idx = np.empty((nrows, k), dtype=np.int32)
    d2 = np.empty((nrows, k), dtype=np.float32)
    if qry is None:
        rc = fn(_ptr(pos), n, _ptr(b), int(k), _ptr(r), nrows, _ptr(idx), _ptr(d2), int(threads or 0), *extra)
    else:
        rc = fn(_ptr(pos), n, _ptr(qry), _ptr(b), int(k), _ptr(r), nrows, _ptr(idx), _ptr(d2), int(threads or 0),
                *extra)
    if rc != 0:
        raise ValueError(f"oracle returned status {rc} (n={n}, k={k})")
    return idx, d2


def knn_brute(pos, k: int, box=None, rows=None, threads: int | None = None, queries=None):
    """O(N^2) definition. Returns (idx int32 [m,k], d2 float32 [m,k]).

    queries=None: self-query. Otherwise row i answers queries[i] against
    the sources `pos` (separate query points)."""
    lib = _load()
    if queries is None:
        return _run(lib.oracle_knn_brute, pos, k, box, rows, threads)
    return _run(lib.oracle_knn_brute_q, pos, k, box, rows, threads, queries=queries)


def knn_grid(pos, k: int, box=None, rows=None, threads: int | None = None, per_cell: float = 2.0, queries=None):
    """Uniform-grid shell search, same bits as knn_brute."""
    lib = _load()
    if queries is None:
        return _run(lib.oracle_knn_grid, pos, k, box, rows, threads, ctypes.c_double(per_cell))
    return _run(lib.oracle_knn_grid_q, pos, k, box, rows, threads, ctypes.c_double(per_cell), queries=queries)


def pair_d2(a, b, box=None):
    """Canonical FP32 d2 for explicit pairs a[i], b[i]."""
    a, bx = _prep(a, box)
    b = np.ascontiguousarray(b, dtype=np.float32)
    out = np.empty(a.shape[0], dtype=np.float32)
    _load().oracle_pair_d2(_ptr(a), _ptr(b), a.shape[0], _ptr(bx), _ptr(out))
    return out


# ----------------------------------------------------------------------------- friends-of-friends
def fof_b2(r_link) -> np.float32:
    """The linking threshold on the canonical d2: RN32(r_link * r_link) (R21)."""
    r = np.float32(r_link)
    return np.float32(r * r)


def fof_labels(pos, r_link, box=None, method: str = "grid"):
    """PAPER.md §5 (L466-474): label[i] = smallest index of i's connected component of the graph
    {i ~ j : canonical d2(p_i, p_j) <= RN32(r_link^2)}."""
    pos, b = _prep(pos, box)
    n = pos.shape[0]
    lab = np.empty(n, dtype=np.int32)
    fn = _load().oracle_fof_grid if method == "grid" else _load().oracle_fof_brute
    rc = fn(_ptr(pos), n, _ptr(b), ctypes.c_float(fof_b2(r_link)), _ptr(lab))
    if rc != 0:
        raise ValueError(f"oracle fof returned status {rc}")
    return lab


def fof_catalogue(pos, labels, box=None, min_count: int = 20):
    """PAPER.md L500-504 summary statistics of the groups with >= min_count points, ordered by
    label (R22): (label int32, count int64, centre of mass float64 [g,3], inertia radius
    float64 [g]). Positions are taken relative to the group's label point, as minimal images when
    periodic; the centre of mass is wrapped into [0, L)."""
    pos = np.asarray(pos, dtype=np.float32).astype(np.float64)
    labels = np.asarray(labels)
    u, cnt = np.unique(labels, return_counts=True)
    keep = cnt >= min_count
    u, cnt = u[keep], cnt[keep]
    L = None if box is None else np.broadcast_to(np.asarray(box, np.float64), (3,))
    com = np.empty((len(u), 3))
    rad = np.empty(len(u))
    for gi, g in enumerate(u):
        m = pos[labels == g]
        disp = m - pos[g]
        if L is not None:
            disp = disp - L * np.round(disp / L)
        mean = disp.mean(axis=0)
        c = pos[g] + mean
        if L is not None:
            c = c - L * np.floor(c / L)
        com[gi] = c
        rad[gi] = np.sqrt(((disp - mean) ** 2).sum(axis=1).mean())
    return u.astype(np.int32), cnt.astype(np.int64), com, rad
