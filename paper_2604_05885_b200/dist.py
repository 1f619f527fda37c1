"""Multi-GPU exact kNN through the library (PAPER.md L112-114
sample-splitter partition, L388-393 distributed kNN, L458 z-order output).

Argument marshalling only: the whole distributed algorithm -- global key frame, sampled
splitters, Morton-range all-to-all-v, local tree and walk, query boxes from the local k-th
distances, ghost exchange, re-walk of the reached queries, reverse exchange to input order --
runs inside libjzknn.so (jz_knn_build_dist / jz_knn_query_dist, csrc/jz_dist.cu) on a jz_comm:

  * NCCL (`Comm.from_torch()`): rank 0 draws the NCCL unique id (jz_comm_unique_id), the id is
    broadcast with torch.distributed (bootstrap plumbing only), every rank calls jz_comm_init on
    its current CUDA device;
  * logical ranks on one device (`LocalWorld`, `run_ranks_simulated`): R host threads, each with
    its own stream, exchange through the library's in-process communicator.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _binding as B


class Comm:
    """A jz_comm (owned)."""

    def __init__(self, handle: ctypes.c_void_p, keep=None):
        self.h = handle
        self._keep = keep  # the local world a logical-rank communicator belongs to
        r, s = ctypes.c_int32(), ctypes.c_int32()
        B.check(B.lib().jz_comm_rank_size(self.h, ctypes.byref(r), ctypes.byref(s)))
        self.rank, self.size = r.value, s.value

    @classmethod
    def from_torch(cls, group=None):
        """NCCL communicator over the ranks of a torch.distributed group (bootstrap: the NCCL
        unique id of rank 0 is broadcast with torch.distributed)."""
        import torch.distributed as dist

        rank, size = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            B.check(B.lib().jz_comm_unique_id(uid))
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        h = ctypes.c_void_p()
        B.check(B.lib().jz_comm_init(uid, size, rank, ctypes.byref(h)))
        return cls(h)

    def free(self):
        if self.h:
            B.lib().jz_comm_free(self.h)
            self.h = None


class LocalWorld:
    """R logical ranks on the current device (jz_comm_local_world)."""

    def __init__(self, R: int):
        self.h = ctypes.c_void_p()
        B.check(B.lib().jz_comm_local_world(int(R), ctypes.byref(self.h)))
        self.size = R

    def comm(self, rank: int) -> Comm:
        h = ctypes.c_void_p()
        B.check(B.lib().jz_comm_init_local(self.h, int(rank), ctypes.byref(h)))
        return Comm(h, keep=self)

    def free(self):
        if self.h:
            B.lib().jz_comm_world_free(self.h)
            self.h = None


def dist_knn(pos: torch.Tensor, gidx_base: int, k: int, box, comm: Comm, order: str = "z", params=None,
             stream=None, stats: dict | None = None):
    """Exact kNN of this rank's input slice against the union over all ranks (collective).

    pos: this rank's CUDA float32 [n, 3] points, global ids gidx_base + i.
    order="z": (idx [m, k], d2 [m, k], row_gidx [m]) for the m points this rank owns after the
    Morton-range partition, in z order. order="input" (F2): the rows of the own input
    slice in input order (row_gidx = gidx_base + arange(n); slices contiguous in rank order)."""
    if order not in ("z", "input"):
        raise ValueError("order must be 'z' or 'input'")
    if not (isinstance(pos, torch.Tensor) and pos.is_cuda and pos.dtype == torch.float32 and pos.dim() == 2
            and pos.shape[1] == 3):
        raise TypeError("pos must be a CUDA float32 [n, 3] tensor")
    L = B.lib()
    pos = pos.contiguous()
    st = B.stream_ptr(stream)
    prm = B.make_params(params)
    ix = ctypes.c_void_p()
    B.check(L.jz_knn_build_dist(comm.h, B.dptr(pos) if pos.shape[0] else None, pos.shape[0], int(gidx_base),
                                B.box3(box), ctypes.byref(prm), st, ctypes.byref(ix)))
    try:
        o = B.JZ_ORDER_Z if order == "z" else B.JZ_ORDER_INPUT
        m = ctypes.c_int64()
        B.check(L.jz_knn_rows_dist(ix, o, ctypes.byref(m)))
        m = m.value
        idx = torch.empty((m, k), dtype=torch.int32, device=pos.device)
        d2 = torch.empty((m, k), dtype=torch.float32, device=pos.device)
        rowg = torch.empty((m,), dtype=torch.int32, device=pos.device)
        B.check(L.jz_knn_query_dist(ix, int(k), o, B.dptr(idx) if m else None, B.dptr(d2) if m else None,
                                    B.dptr(rowg) if m else None, st))
        if stats is not None:
            c = (ctypes.c_int64 * 4)()
            t = (ctypes.c_double * 6)()
            B.check(L.jz_knn_dist_stats(ix, c, t))
            stats.update({"n_local": c[0], "n_ghost": c[1], "n_requery": c[2], "n_qbox": c[3],
                          "ms": {"partition": t[0], "local_build": t[1], "local_walk": t[2], "ghosts_rewalk": t[3],
                                 "reverse": t[4]}, "busy_ms_total": t[5]})
    finally:
        L.jz_knn_free(ix)
    return idx, d2, rowg


def run_ranks_simulated(pos_np: np.ndarray, k: int, box, R: int, params=None, order: str = "z",
                        stats: list | None = None):
    """R logical ranks on the current CUDA device (threads, each with its own stream), each owning
    a contiguous input slice. Returns the gathered rows as full arrays in input order and the
    number of rows each rank returned."""
    n = pos_np.shape[0]
    bounds = [(n * i) // R for i in range(R + 1)]
    world = LocalWorld(R)
    comms = [world.comm(r) for r in range(R)]
    res = [None] * R
    err = []

    def work(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                p = torch.from_numpy(np.ascontiguousarray(pos_np[bounds[r]:bounds[r + 1]])).cuda()
                sd = {} if stats is not None else None
                out = dist_knn(p, bounds[r], k, box, comms[r], order=order, params=params, stream=st, stats=sd)
                st.synchronize()
                res[r] = out  # copied to the host after every rank finished (pageable copies serialise)
                if stats is not None:
                    stats.append((r, sd))
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)

    ths = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    for c in comms:
        c.free()
    world.free()
    if err:
        raise err[0]
    res = [tuple(x.cpu().numpy() for x in out) for out in res]
    idx = np.empty((n, k), np.int32)
    d2 = np.empty((n, k), np.float32)
    seen = np.zeros(n, bool)
    for (i, d, g) in res:
        idx[g] = i
        d2[g] = d
        seen[g] = True
    assert seen.all(), "some rows were not produced"
    return idx, d2, [r[0].shape[0] for r in res]
