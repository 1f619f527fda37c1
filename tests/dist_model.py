"""CPU model of the library's distributed kNN (TEST INFRASTRUCTURE ONLY).

The product path is jz_knn_build_dist / jz_knn_query_dist inside libjzknn.so (jz_dist.cu) on a
jz_comm. This module restates the same protocol step by step over torch.distributed (gloo, CPU)
with the numpy stand-ins of tests/cpu_backend.py, so the world-size-2/3 tests check the
partition + ghost protocol itself on CPU:
  1. frame (all-reduced bbox when open), 2. sampled splitters, 3. Morton-range exchange,
  4. local rows (exact over the local points: their k-th d2 bounds the global one),
  5. query boxes (AABB + largest local k-th d2) all-gathered, 6. ghosts = points within a peer
  box's radius, plus the boxes they reached (all-reduced), 7. queries of reached boxes re-walked
  over local + ghost points, 8. optional reverse exchange to input order (F2).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import knn_brute


class TorchComm:
    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_gather_v(self, t):
        d = self.dist
        n = torch.tensor([t.shape[0]], dtype=torch.int64)
        ns = [torch.zeros_like(n) for _ in range(self.size)]
        d.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        m = max(ns) if ns else 0
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.size)]
        d.all_gather(outs, pad, group=self.group)
        return [o[:c] for o, c in zip(outs, ns)]

    def all_to_all_v(self, send, send_counts, recv_counts):
        recv = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype)
        self.dist.all_to_all_single(recv, send, output_split_sizes=list(recv_counts),
                                    input_split_sizes=list(send_counts), group=self.group)
        return recv

    def all_to_all_counts(self, counts):
        s = torch.tensor(counts, dtype=torch.int64)
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s, group=self.group)
        return [int(x) for x in r.tolist()]

    def all_reduce(self, t, op):
        self.dist.all_reduce(t, op=op, group=self.group)
        return t


def splitters_from_samples(all_samples: torch.Tensor, R: int) -> torch.Tensor:
    """R - 1 quantile splitters spl[i-1] = sorted[(i m) / R], as k_splitters."""
    s = torch.sort(all_samples).values
    m = s.shape[0]
    if m == 0 or R == 1:
        return s[:0]
    return s[torch.tensor([(i * m) // R for i in range(1, R)], dtype=torch.int64)].contiguous()


def dist_knn_model(pos, gidx_base, k, box, comm, be, n_samp=64, seed=0, order="z"):
    import torch.distributed as dist

    R, r = comm.size, comm.rank
    if box is not None:
        frame = {"box": box}
    else:
        lo, hi = be.bbox(pos)
        lo = comm.all_reduce(lo.clone(), dist.ReduceOp.MIN)
        hi = comm.all_reduce(hi.clone(), dist.ReduceOp.MAX)
        ln, hn = lo.numpy().astype(np.float32), hi.numpy().astype(np.float32)
        ext = float(max(np.float32(hn[d] - ln[d]) for d in range(3)))
        frame = {"box": None, "origin": [float(x) for x in ln], "extent": ext if ext > 0 else 1.0}
    keys = be.morton_keys(pos, frame)
    samp = be.sample(keys, n_samp, seed * 1000003 + r)
    spl = splitters_from_samples(torch.cat(comm.all_gather_v(samp)), R)
    dest, counts = be.bucket(keys, spl)
    local = comm.all_to_all_v(be.pack(pos, gidx_base, dest, counts), counts, comm.all_to_all_counts(counts))
    m = local.shape[0]
    ix = be.build(local, m, box)
    # 4. local rows (exact over the local points)
    if m >= k:
        idx, d2, rowg = be.query_z(ix, k)
    else:
        idx = torch.zeros((m, k), dtype=torch.int32)
        d2 = torch.zeros((m, k), dtype=torch.float32)
        rowg = torch.from_numpy(ix.pts4[:, 3].view(np.int32).copy())
    if R > 1:
        # 5. query boxes from the local k-th d2 (chunks of the z order); +inf without local rows
        qb, members = be.query_boxes(ix, k, r, d2 if m >= k else None)
        allb = comm.all_gather_v(qb)
        boff = np.concatenate([[0], np.cumsum([b.shape[0] for b in allb])]).astype(int)
        allb = torch.cat(allb) if allb else qb
        # 6. ghosts + the boxes they reached
        mask, gcounts, hit = be.select_ghosts(ix, allb, r, R)
        gsend = be.pack_ghosts(ix, mask, gcounts)
        ghosts = comm.all_to_all_v(gsend, gcounts, comm.all_to_all_counts(gcounts))
        hit = comm.all_reduce(torch.from_numpy(hit.astype(np.int32)), dist.ReduceOp.MAX).numpy()
        # 7. re-walk the queries of my reached boxes over local + ghost points
        mine = hit[boff[r]:boff[r + 1]]
        sel = np.concatenate([members[j] for j in range(len(members)) if mine[j]] + [np.zeros(0, np.int64)])
        sel = np.sort(sel).astype(np.int64)
        if m > 0 and ghosts.shape[0] > 0 and sel.size:
            allp = np.concatenate([ix.pts4, ghosts.numpy()]).astype(np.float32)
            g = allp[:, 3].view(np.int32)
            i2, dd2 = knn_brute(allp[:, :3], k, box, rows=sel)
            idx = idx.clone()
            d2 = d2.clone()
            idx[torch.from_numpy(sel)] = torch.from_numpy(g[i2])
            d2[torch.from_numpy(sel)] = torch.from_numpy(dd2)
        assert m < k and sel.size == m or m >= k, "a rank without local rows must re-walk every query"
    if order == "input":
        return _to_input_order(idx, d2, rowg, pos.shape[0], gidx_base, k, comm, be)
    return idx, d2, rowg


def _to_input_order(idx, d2, rowg, n_own, gidx_base, k, comm, be):
    R = comm.size
    sizes = comm.all_gather_v(torch.tensor([[n_own, gidx_base]], dtype=torch.int64))
    bounds = np.concatenate([[0], np.cumsum([int(s[0, 0]) for s in sizes])])
    spl = torch.tensor(bounds[1:R], dtype=torch.int64)
    dest, counts = be.bucket(rowg.to(torch.int64), spl)
    recv = comm.all_to_all_v(be.pack_rows(idx, d2, rowg, dest, counts), counts, comm.all_to_all_counts(counts))
    assert recv.shape[0] == n_own
    oi, od = be.scatter_rows(recv, k, gidx_base, n_own, None)
    return oi, od, torch.arange(gidx_base, gidx_base + n_own, dtype=torch.int32)
