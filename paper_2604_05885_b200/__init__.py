"""B200-native exact k-nearest-neighbour search on a Morton plane hierarchy
(jz-tree, arXiv 2604.05885) -- Python front end of libjzknn.so.

    import torch, paper_2604_05885_b200 as jz
    pos = torch.rand(10**6, 3, device="cuda")
    idx, d2 = jz.knn(pos, k=16, box=1.0)          # rows in input order

    ix = jz.KnnIndex(pos, box=1.0)                 # build once (§2)
    idx, d2 = ix.query(16)                         # query many k (§3)
    idx, d2, gidx = ix.query(16, order="z")        # z-order rows + their global ids
    idx, d2 = jz.knn(src, k=16, queries=qry)       # separate query points
    idx, d2 = ix.query(100)                        # k > 32: ceil(k/32) LeafToLeaf passes

All compute runs in the library's sm_100a kernels; PyTorch only provides device
memory and the stream. See include/jz_knn.h for the C ABI.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _binding as B
from ._binding import JzError, JZ_FLAG_FRAME, JZ_FLAG_NO_EARLY_EXIT, JZ_FLAG_NO_SEGSORT  # noqa: F401

__all__ = ["KnnIndex", "knn", "knn_host", "JzError", "set_timing"]


def set_timing(on: bool = True):
    B.lib().jz_set_timing(1 if on else 0)


class KnnIndex:
    """Tree over `pos` (CUDA float32 [n,3], or [n,4] {x,y,z,bits(gidx)} with n_query; a
    negative gidx marks a query-only point). With `queries` ([m,3]) the tree is built jointly
    over sources `pos` and the queries and row i answers queries[i]."""

    def __init__(self, pos: torch.Tensor, box=None, params=None, n_query: int | None = None, stream=None,
                 queries: torch.Tensor | None = None):
        if not (isinstance(pos, torch.Tensor) and pos.is_cuda and pos.dtype == torch.float32):
            raise TypeError("pos must be a CUDA float32 tensor")
        pos = pos.contiguous()
        self._lib = B.lib()
        self._h = ctypes.c_void_p()
        self.box = box
        self.stream = stream
        prm = B.make_params(params)
        st = B.stream_ptr(stream)
        if queries is not None:
            if not (isinstance(queries, torch.Tensor) and queries.is_cuda and queries.dtype == torch.float32
                    and queries.dim() == 2 and queries.shape[1] == 3 and pos.dim() == 2 and pos.shape[1] == 3):
                raise TypeError("pos and queries must be CUDA float32 [n,3] tensors")
            if n_query is not None:
                raise ValueError("n_query and queries are exclusive")
            queries = queries.contiguous()
            B.check(self._lib.jz_knn_build_xq(B.dptr(pos), pos.shape[0], B.dptr(queries), queries.shape[0],
                                              B.box3(box), ctypes.byref(prm), st, ctypes.byref(self._h)))
        elif pos.dim() == 2 and pos.shape[1] == 3:
            if n_query is not None and n_query != pos.shape[0]:
                raise ValueError("n_query needs [n,4] xyzg input")
            B.check(self._lib.jz_knn_build(B.dptr(pos), pos.shape[0], B.box3(box), ctypes.byref(prm), st,
                                           ctypes.byref(self._h)))
        elif pos.dim() == 2 and pos.shape[1] == 4:
            nq = pos.shape[0] if n_query is None else int(n_query)
            B.check(self._lib.jz_knn_build_xyzg(B.dptr(pos), pos.shape[0], nq, B.box3(box), ctypes.byref(prm), st,
                                                ctypes.byref(self._h)))
        else:
            raise ValueError("pos must be [n,3] or [n,4]")
        self.n = pos.shape[0]
        self.device = pos.device
        m = ctypes.c_int64()
        B.check(self._lib.jz_knn_rows(self._h, ctypes.byref(m)))
        self.rows = m.value

    def query(self, k: int, order: str = "input", out=None):
        """k nearest neighbours of every query point: (idx int32 [m,k], d2 float32 [m,k])
        (+ row gidx int32 [m] for order="z")."""
        o = {"input": B.JZ_ORDER_INPUT, "z": B.JZ_ORDER_Z}[order]
        if out is None:
            idx = torch.empty((self.rows, k), dtype=torch.int32, device=self.device)
            d2 = torch.empty((self.rows, k), dtype=torch.float32, device=self.device)
            rg = torch.empty((self.rows,), dtype=torch.int32, device=self.device) if o == B.JZ_ORDER_Z else None
        else:
            idx, d2, rg = out
        B.check(self._lib.jz_knn_query(self._h, int(k), o, B.dptr(idx), B.dptr(d2),
                                       B.dptr(rg) if rg is not None else None, B.stream_ptr(self.stream)))
        return (idx, d2) if o == B.JZ_ORDER_INPUT else (idx, d2, rg)

    def fof(self, r_link: float, min_count: int = 20, labels=None):
        """Friends-of-friends (§5): (labels int32 [n] in input order = smallest
        input index of each point's group, catalogue dict of the groups with >= min_count points
        in the paper's group order: label, count, com [g,3] float64, rad float64)."""
        if labels is None:
            labels = torch.empty((self.n,), dtype=torch.int32, device=self.device)
        ng = ctypes.c_int64()
        st = B.stream_ptr(self.stream)
        B.check(self._lib.jz_fof(self._h, float(r_link), int(min_count), B.dptr(labels), ctypes.byref(ng), st))
        g = ng.value
        cat = {"label": torch.empty((g,), dtype=torch.int32, device=self.device),
               "count": torch.empty((g,), dtype=torch.int32, device=self.device),
               "com": torch.empty((g, 3), dtype=torch.float64, device=self.device),
               "rad": torch.empty((g,), dtype=torch.float64, device=self.device)}
        if g:
            B.check(self._lib.jz_fof_catalogue(self._h, g, B.dptr(cat["label"]), B.dptr(cat["count"]),
                                               B.dptr(cat["com"]), B.dptr(cat["rad"]), st))
        return labels, cat

    def fof_group_order(self):
        """Group order of the last fof(): (order int32 [n] = input rows with every
        group contiguous, groups in z order of their roots, z order inside; group_beg int32
        [ngroups + 1] block starts)."""
        order = torch.empty((self.n,), dtype=torch.int32, device=self.device)
        beg = torch.empty((self.n + 1,), dtype=torch.int32, device=self.device)
        ng = ctypes.c_int64()
        B.check(self._lib.jz_fof_group_order(self._h, B.dptr(order), B.dptr(beg), ctypes.byref(ng),
                                             B.stream_ptr(self.stream)))
        return order, beg[: ng.value + 1]

    def stage_times(self):
        """Per-phase device ms of the last build + query (needs set_timing(True) before the build)."""
        t = (ctypes.c_float * 6)()
        ev = ctypes.c_int64()
        B.check(self._lib.jz_knn_stage_times(self._h, t, ctypes.byref(ev)))
        names = ["frame", "sort", "tree", "node2node", "leaf2leaf", "total"]
        d = {n: float(v) for n, v in zip(names, t)}
        d["evals"] = ev.value
        st = (ctypes.c_int64 * 9)()
        B.check(self._lib.jz_knn_stats(self._h, st))
        d["inserts"], d["leaves"], d["planes"] = st[1], st[2], st[3]
        d["walk"] = {"appends": st[4], "merge_rounds": st[5], "compactions": st[6], "leaves_staged": st[7], "items": st[8]}
        return d

    # ---- introspection (tests)
    def _copy(self, what, plane=0, dtype=np.uint8):
        nbytes = self._lib.jz_knn_debug_copy(self._h, what, plane, None, 0)
        if nbytes < 0:
            raise ValueError("bad introspection request")
        buf = np.empty(nbytes, dtype=np.uint8)
        if nbytes:
            self._lib.jz_knn_debug_copy(self._h, what, plane, buf.ctypes.data_as(ctypes.c_void_p), nbytes)
        return buf.view(dtype)

    def sorted_keys(self):
        return self._copy(0, dtype=np.uint64)

    def sorted_points(self):
        return self._copy(1, dtype=np.float32).reshape(-1, 4)

    def perm(self):
        return self._copy(2, dtype=np.int32)

    def num_planes(self):
        return int(self._copy(5, dtype=np.int64)[0])

    def plane_beg(self, p):
        return self._copy(3, p, dtype=np.int32)

    def plane_boxes(self, p):
        return self._copy(4, p, dtype=np.float32).reshape(-1, 8)

    def handle(self):
        return self._h

    def free(self):
        if self._h:
            self._lib.jz_knn_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def knn(pos: torch.Tensor, k: int, box=None, order: str = "input", params=None, stream=None, queries=None):
    """Exact kNN of every point of `pos` among all points (self included), or of every row of
    `queries` among the points of `pos`."""
    ix = KnnIndex(pos, box=box, params=params, stream=stream, queries=queries)
    try:
        return ix.query(k, order=order)
    finally:
        ix.free()


def fof(pos: torch.Tensor, r_link: float, box=None, min_count: int = 20, params=None, stream=None):
    """One-shot friends-of-friends (build + jz_fof): (labels, catalogue), see KnnIndex.fof."""
    ix = KnnIndex(pos, box=box, params=params, stream=stream)
    try:
        return ix.fof(r_link, min_count)
    finally:
        ix.free()


def knn_host_z(pos: np.ndarray, k: int, box=None, params=None, out=None, stream=None):
    """End to end on host arrays with z-order rows streamed to the host during the walk
    (jz_knn_search_host_z): (idx [n, k], d2 [n, k], row_gidx [n])."""
    pos = np.ascontiguousarray(pos, dtype=np.float32)
    n = pos.shape[0]
    if out is None:
        out = (np.empty((n, k), dtype=np.int32), np.empty((n, k), dtype=np.float32), np.empty(n, dtype=np.int32))
    idx, d2, rg = out
    prm = B.make_params(params)
    B.check(B.lib().jz_knn_search_host_z(pos.ctypes.data_as(ctypes.c_void_p), n, B.box3(box), ctypes.byref(prm),
                                         int(k), idx.ctypes.data_as(ctypes.c_void_p),
                                         d2.ctypes.data_as(ctypes.c_void_p), rg.ctypes.data_as(ctypes.c_void_p),
                                         B.stream_ptr(stream)))
    return idx, d2, rg


def knn_host(pos: np.ndarray, k: int, box=None, params=None, out=None, stream=None):
    """End to end on host arrays through jz_knn_search_host (H2D, build, query, D2H)."""
    pos = np.ascontiguousarray(pos, dtype=np.float32)
    n = pos.shape[0]
    if out is None:
        idx = np.empty((n, k), dtype=np.int32)
        d2 = np.empty((n, k), dtype=np.float32)
    else:
        idx, d2 = out
    prm = B.make_params(params)
    B.check(B.lib().jz_knn_search_host(pos.ctypes.data_as(ctypes.c_void_p), n, B.box3(box), ctypes.byref(prm),
                                       int(k), idx.ctypes.data_as(ctypes.c_void_p),
                                       d2.ctypes.data_as(ctypes.c_void_p), B.stream_ptr(stream)))
    return idx, d2
