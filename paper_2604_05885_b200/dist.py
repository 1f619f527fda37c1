"""Multi-GPU exact kNN: Morton-range partition + ghost exchange (PAPER.md
L112-114 sample-based splitters, L388-393 distributed kNN, L458 z-order output).

One process per GPU. The per-rank compute runs in the library's kernels (a `Backend`); the
exchanges are collectives on a `Comm` (torch.distributed over NCCL on B200s, gloo in CPU
tests, or an in-process simulation that runs R logical ranks on one device). Steps:

  1. key frame: periodic box (every rank identical), or all-reduced bounding box (open)
  2. each rank draws N_samp = 1000 keys; all-gather; every rank sorts the R * N_samp
     samples identically and takes R - 1 quantiles as splitters (no broadcast needed)
  3. bucket points by splitter (a key equal to a splitter goes to the upper rank), exchange
     counts, all-to-all-v of float4 {x, y, z, bits(gidx)} rows
  4. local tree over the received points; NodeToNode walk to the leaf plane gives R_max^2
     per leaf, which bounds every local query's k-th distance (a rank holding >= k points
     has >= k candidates within it; ghosts can only shrink the k-th distance)
  5. query boxes (plane nodes: AABB + max R_max^2) all-gathered; each rank flags the local
     points reachable from a peer's box (exact box bound), exchanges counts, all-to-all-v
     of ghost rows
  6. final tree over local + ghost points, queries = local points only; rows in z-order
     with their global indices
  7. (order="input") reverse all-to-all-v: every row goes to the rank owning its
     input row (splitters = the input-slice bounds), which writes it at gidx - base
     (the paper's "final reordering step")

Correctness does not depend on the partition: any point within a query's true k-th radius
is either local or flagged as a ghost for that query's rank.
"""
from __future__ import annotations

import threading
import time

import numpy as np
import torch

N_SAMP = 1000
QBOX_NODES = int(__import__('os').environ.get('JZ_QBOX_NODES', '4096'))  # query-box plane size cap


# ----------------------------------------------------------------------------- comms
class Comm:
    rank: int
    size: int

    def all_gather_v(self, t: torch.Tensor) -> list:
        """Gather tensors of varying first dimension from all ranks (same dtype/trailing dims)."""
        raise NotImplementedError

    def all_to_all_v(self, send: torch.Tensor, send_counts: list, recv_counts: list) -> torch.Tensor:
        raise NotImplementedError

    def all_to_all_counts(self, counts: list) -> list:
        raise NotImplementedError

    def all_reduce_minmax(self, lo: torch.Tensor, hi: torch.Tensor):
        raise NotImplementedError

    def max_scalar(self, v: float) -> float:
        raise NotImplementedError

    def barrier(self):
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_gather_v(self, t):
        d = self.dist
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = [torch.zeros_like(n) for _ in range(self.size)]
        d.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        m = max(ns) if ns else 0
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.size)]
        d.all_gather(outs, pad, group=self.group)
        return [o[:c] for o, c in zip(outs, ns)]

    def all_to_all_v(self, send, send_counts, recv_counts):
        recv = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, output_split_sizes=list(recv_counts),
                                    input_split_sizes=list(send_counts), group=self.group)
        return recv

    def all_to_all_counts(self, counts):
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        s = torch.tensor(counts, dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s, group=self.group)
        return [int(x) for x in r.tolist()]

    def all_reduce_minmax(self, lo, hi):
        self.dist.all_reduce(lo, op=self.dist.ReduceOp.MIN, group=self.group)
        self.dist.all_reduce(hi, op=self.dist.ReduceOp.MAX, group=self.group)
        return lo, hi

    def max_scalar(self, v):
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)


class SimWorld:
    """R logical ranks in one process (threads), exchanging through shared Python lists."""

    def __init__(self, size):
        self.size = size
        self._bar = threading.Barrier(size)
        self._slots = [None] * size

    def exchange(self, rank, obj):
        self._slots[rank] = obj
        self._bar.wait()
        out = list(self._slots)
        self._bar.wait()
        return out


class SimComm(Comm):
    def __init__(self, world: SimWorld, rank: int):
        self.w = world
        self.rank = rank
        self.size = world.size

    def all_gather_v(self, t):
        return [x.clone() for x in self.w.exchange(self.rank, t)]

    def all_to_all_v(self, send, send_counts, recv_counts):
        off = np.concatenate([[0], np.cumsum(send_counts)]).astype(int)
        parts = [send[off[i]:off[i + 1]] for i in range(self.size)]
        allp = self.w.exchange(self.rank, parts)
        got = [allp[src][self.rank] for src in range(self.size)]
        out = torch.cat(got) if got else send[:0]
        assert out.shape[0] == sum(recv_counts)
        return out

    def all_to_all_counts(self, counts):
        allc = self.w.exchange(self.rank, list(counts))
        return [allc[src][self.rank] for src in range(self.size)]

    def all_reduce_minmax(self, lo, hi):
        al = self.w.exchange(self.rank, (lo.clone(), hi.clone()))
        return torch.stack([a[0] for a in al]).min(0).values, torch.stack([a[1] for a in al]).max(0).values

    def max_scalar(self, v):
        return max(self.w.exchange(self.rank, v))

    def barrier(self):
        self.w.exchange(self.rank, None)


# ----------------------------------------------------------------------------- GPU backend
class GpuBackend:
    """Per-rank compute through the C ABI (all steps are library kernels)."""

    def __init__(self, params=None, stream=None, stats=None):
        from . import _binding as B

        self.stats = stats
        self.B = B
        self.lib = B.lib()
        self.params = params
        self.stream = stream

    def _st(self):
        return self.B.stream_ptr(self.stream)

    def morton_keys(self, pos, frame):
        import ctypes

        keys = torch.empty(pos.shape[0], dtype=torch.int64, device=pos.device)
        if frame["box"] is not None:
            self.B.check(self.lib.jz_morton_keys(self.B.dptr(pos), pos.shape[0], self.B.box3(frame["box"]), None, 0.0,
                                                 self.B.dptr(keys), self._st()))
        else:
            org = (ctypes.c_float * 3)(*frame["origin"])
            self.B.check(self.lib.jz_morton_keys(self.B.dptr(pos), pos.shape[0], None, org, float(frame["extent"]),
                                                 self.B.dptr(keys), self._st()))
        return keys

    def bbox(self, pos):
        return pos.min(0).values.clone(), pos.max(0).values.clone()

    def sample(self, keys, n, seed):
        if keys.shape[0] == 0:
            return keys[:0]
        g = torch.Generator(device="cpu").manual_seed(seed)
        sel = torch.randint(0, keys.shape[0], (n,), generator=g).to(keys.device)
        return keys[sel]

    def sort_samples(self, s):
        return torch.sort(s).values

    def bucket(self, keys, splitters):
        R = splitters.shape[0] + 1
        dest = torch.empty(keys.shape[0], dtype=torch.int32, device=keys.device)
        counts = torch.empty(R, dtype=torch.int64, device=keys.device)
        self.B.check(self.lib.jz_bucket_by_splitters(self.B.dptr(keys), keys.shape[0], self.B.dptr(splitters),
                                                     splitters.shape[0], self.B.dptr(dest), self.B.dptr(counts),
                                                     self._st()))
        return dest, [int(c) for c in counts.tolist()]

    def pack(self, pos, gbase, dest, counts):
        R = len(counts)
        off = torch.tensor(np.concatenate([[0], np.cumsum(counts)[:-1]]), dtype=torch.int64, device=pos.device)
        out = torch.empty((pos.shape[0], 4), dtype=torch.float32, device=pos.device)
        self.B.check(self.lib.jz_pack_by_rank(self.B.dptr(pos), pos.shape[0], int(gbase), self.B.dptr(dest),
                                              self.B.dptr(off), R, self.B.dptr(out), self._st()))
        return out

    def build(self, pts4, n_query, box):
        from . import KnnIndex

        return KnnIndex(pts4, box=box, params=self.params, n_query=n_query, stream=self.stream)

    def query_boxes(self, ix, k, rank):
        import ctypes

        # finest plane with at most QBOX_NODES nodes (peers test every box against their top nodes)
        nn = ctypes.c_int64()
        P = ix.num_planes()
        plane = P - 1
        for p in range(P):
            self.B.check(self.lib.jz_knn_plane_nodes(ix.handle(), p, ctypes.byref(nn)))
            if nn.value <= QBOX_NODES:
                plane = p
                break
        self.B.check(self.lib.jz_knn_plane_nodes(ix.handle(), plane, ctypes.byref(nn)))
        boxes = torch.empty((nn.value, 8), dtype=torch.float32, device=ix.device)
        if k > ix.n:
            k_eff = max(1, min(k, ix.n))
        else:
            k_eff = k
        self.B.check(self.lib.jz_knn_query_boxes(ix.handle(), int(k_eff), plane, int(rank), self.B.dptr(boxes),
                                                 self._st()))
        if k > ix.n:  # fewer than k local points: no finite bound
            boxes[:, 3] = float("inf")
        return boxes

    def select_ghosts(self, ix, boxes, rank, R):
        mask = torch.empty(ix.n, dtype=torch.int32, device=ix.device)
        counts = torch.empty(R, dtype=torch.int64, device=ix.device)
        self.B.check(self.lib.jz_knn_select_ghosts(ix.handle(), self.B.dptr(boxes), boxes.shape[0], int(rank), R,
                                                   self.B.dptr(mask), self.B.dptr(counts), self._st()))
        return mask, [int(c) for c in counts.tolist()]

    def pack_ghosts(self, ix, mask, counts):
        R = len(counts)
        off = torch.tensor(np.concatenate([[0], np.cumsum(counts)[:-1]]), dtype=torch.int64, device=ix.device)
        out = torch.empty((max(1, sum(counts)), 4), dtype=torch.float32, device=ix.device)
        self.B.check(self.lib.jz_knn_pack_ghosts(ix.handle(), self.B.dptr(mask), R, self.B.dptr(off),
                                                 self.B.dptr(out), self._st()))
        return out[: sum(counts)]

    def query_z(self, ix, k):
        out = ix.query(k, order="z")
        if self.stats is not None:  # LeafToLeaf time / evaluations of the final walk (bench roofline)
            t = ix.stage_times()
            self.stats["leaf2leaf_ms"] = t["leaf2leaf"]
            self.stats["evals"] = t["evals"]
        return out

    def pack_rows(self, idx, d2, rowg, dest, counts):
        k = idx.shape[1]
        m = idx.shape[0]
        off = torch.tensor(np.concatenate([[0], np.cumsum(counts)[:-1]]), dtype=torch.int64, device=idx.device)
        out = torch.empty((max(1, m), 2 * k + 1), dtype=torch.int32, device=idx.device)
        self.B.check(self.lib.jz_pack_rows(self.B.dptr(idx), self.B.dptr(d2), self.B.dptr(rowg), m, k,
                                           self.B.dptr(dest), self.B.dptr(off), len(counts), self.B.dptr(out),
                                           self._st()))
        return out[:m]

    def scatter_rows(self, rows, k, base, n, device):
        idx = torch.empty((n, k), dtype=torch.int32, device=device)
        d2 = torch.empty((n, k), dtype=torch.float32, device=device)
        self.B.check(self.lib.jz_scatter_rows(self.B.dptr(rows), rows.shape[0], k, int(base), n, self.B.dptr(idx),
                                              self.B.dptr(d2), self._st()))
        return idx, d2

    def free(self, ix):
        ix.free()


# ----------------------------------------------------------------------------- orchestration
def splitters_from_samples(all_samples: torch.Tensor, R: int, sort_fn) -> torch.Tensor:
    """R - 1 quantile splitters of the sorted samples ("the sampled points are evenly
    partitioned")."""
    s = sort_fn(all_samples)
    m = s.shape[0]
    if m == 0 or R == 1:
        return s[:0]
    idx = torch.tensor([(i * m) // R for i in range(1, R)], dtype=torch.int64, device=s.device)
    return s[idx].contiguous()


def dist_knn(pos: torch.Tensor, gidx_base: int, k: int, box, comm: Comm, backend, n_samp: int = N_SAMP,
             seed: int = 0, timings: dict | None = None, order: str = "z"):
    """Exact kNN of this rank's slice against the union over ranks.

    pos: this rank's [n_r, 3] float32 points (global ids gidx_base + i; the slices of the
    ranks are contiguous and in rank order).
    order="z": returns (idx [m, k] int32 global ids, d2 [m, k] float32, row_gidx [m] int32),
    the rows of the points this rank owns after the Morton-range partition, in z-order.
    order="input" (F2): returns the rows of this rank's own input slice, row i = input point
    gidx_base + i (row_gidx = gidx_base + arange(n_r))."""
    if order not in ("z", "input"):
        raise ValueError("order must be 'z' or 'input'")
    R, r = comm.size, comm.rank
    t = timings if timings is not None else {}
    t0 = time.perf_counter()
    # 1. frame
    if box is not None:
        frame = {"box": box}
    else:
        lo, hi = backend.bbox(pos)
        lo, hi = comm.all_reduce_minmax(lo, hi)
        lo_np, hi_np = lo.cpu().numpy().astype(np.float32), hi.cpu().numpy().astype(np.float32)
        ext = float(max(np.float32(hi_np[d] - lo_np[d]) for d in range(3)))
        frame = {"box": None, "origin": [float(x) for x in lo_np], "extent": ext if ext > 0 else 1.0}
    keys = backend.morton_keys(pos, frame)
    if timings is not None:
        torch.cuda.synchronize()
        t["keys"] = time.perf_counter() - t0
    # 2. splitters
    samp = backend.sample(keys, n_samp, seed * 1000003 + r)
    allsamp = torch.cat(comm.all_gather_v(samp))
    spl = splitters_from_samples(allsamp, R, backend.sort_samples)
    # 3. redistribute
    dest, counts = backend.bucket(keys, spl)
    rcounts = comm.all_to_all_counts(counts)
    send = backend.pack(pos, gidx_base, dest, counts)
    local = comm.all_to_all_v(send, counts, rcounts)
    m = local.shape[0]
    t["partition"] = time.perf_counter() - t0
    # 4-5. local tree, query boxes, ghosts
    t1 = time.perf_counter()
    gh_counts = [0] * R
    ghosts = local[:0]
    if R > 1:
        if m > 0:
            ix = backend.build(local, m, box)
            qb = backend.query_boxes(ix, k, r)
        else:
            ix, qb = None, local.new_zeros((0, 8))
        allb = torch.cat(comm.all_gather_v(qb))
        if ix is not None:
            mask, gh_counts = backend.select_ghosts(ix, allb, r, R)
            gsend = backend.pack_ghosts(ix, mask, gh_counts)
        else:
            gsend = local.new_zeros((0, 4))
        grecv = comm.all_to_all_counts(gh_counts)
        ghosts = comm.all_to_all_v(gsend, gh_counts, grecv)
        if ix is not None:
            backend.free(ix)
    t["ghosts"] = time.perf_counter() - t1
    t["n_local"], t["n_ghost"] = m, ghosts.shape[0]
    # 6. final walk over local + ghosts, local queries only
    t2 = time.perf_counter()
    if m == 0:
        z = local.new_zeros((0, k))
        idx, d2, rowg = z.to(torch.int32), z, local.new_zeros((0,), dtype=torch.int32)
        if order == "input":
            return _to_input_order(idx, d2, rowg, pos.shape[0], gidx_base, k, comm, backend)
        return idx, d2, rowg
    allpts = torch.cat([local, ghosts]) if ghosts.shape[0] else local
    if allpts.shape[0] < k:
        raise ValueError("fewer than k points reachable on a rank (k > global n?)")
    ix2 = backend.build(allpts, m, box)
    idx, d2, rowg = backend.query_z(ix2, k)
    backend.free(ix2)
    t["walk"] = time.perf_counter() - t2
    if order == "input":
        t3 = time.perf_counter()
        idx, d2, rowg = _to_input_order(idx, d2, rowg, pos.shape[0], gidx_base, k, comm, backend)
        t["reorder"] = time.perf_counter() - t3
    return idx, d2, rowg


def _to_input_order(idx, d2, rowg, n_own, gidx_base, k, comm, backend):
    """F2: route every z-ordered row to the rank owning its input row and write it there."""
    R = comm.size
    dev = idx.device
    sizes = comm.all_gather_v(torch.tensor([n_own, gidx_base], dtype=torch.int64, device=dev))
    sizes = [(int(x[0]), int(x[1])) for x in sizes]
    bounds = np.concatenate([[0], np.cumsum([c for c, _ in sizes])])
    if any(b != int(bounds[r]) for r, (_, b) in enumerate(sizes)):
        raise ValueError("order='input' needs contiguous input slices in rank order")
    spl = torch.tensor(bounds[1:R], dtype=torch.int64, device=dev)
    dest, counts = backend.bucket(rowg.to(torch.int64), spl)
    rcounts = comm.all_to_all_counts(counts)
    send = backend.pack_rows(idx, d2, rowg, dest, counts)
    recv = comm.all_to_all_v(send, counts, rcounts)
    if recv.shape[0] != n_own:
        raise RuntimeError(f"rank received {recv.shape[0]} rows for {n_own} owned input points")
    oi, od = backend.scatter_rows(recv, k, gidx_base, n_own, dev)
    return oi, od, torch.arange(gidx_base, gidx_base + n_own, dtype=torch.int32, device=dev)


def run_ranks_simulated(pos_np: np.ndarray, k: int, box, R: int, params=None, n_samp: int = N_SAMP,
                        order: str = "z"):
    """Run R logical ranks on the current CUDA device (threads + SimComm), each owning a
    contiguous input slice. Returns the gathered rows as full arrays in input order (with
    order="input" every rank already returns its own slice's rows, F2)."""
    n = pos_np.shape[0]
    bounds = [(n * i) // R for i in range(R + 1)]
    world = SimWorld(R)
    res = [None] * R
    err = []

    def work(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                be = GpuBackend(params=params, stream=st)
                p = torch.from_numpy(np.ascontiguousarray(pos_np[bounds[r]:bounds[r + 1]])).cuda()
                out = dist_knn(p, bounds[r], k, box, SimComm(world, r), be, n_samp=n_samp, order=order)
                st.synchronize()
                res[r] = tuple(x.cpu().numpy() for x in out)
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            world._bar.abort()

    ths = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    if err:
        raise err[0]
    idx = np.empty((n, k), np.int32)
    d2 = np.empty((n, k), np.float32)
    seen = np.zeros(n, bool)
    for (i, d, g) in res:
        idx[g] = i
        d2[g] = d
        seen[g] = True
    assert seen.all(), "some rows were not produced"
    return idx, d2, [r[0].shape[0] for r in res]


# ----------------------------------------------------------------------------- bench (torchrun)
def run_bench_distributed(args, metric, unit):
    """bench.py under torchrun: C4 (10^8 clustered, k = 16) split across ranks (strong scaling).
    Device time per step = max over ranks (CUDA events on each rank's stream); e2e = the same
    with each rank's slice copied from pinned host memory and its rows copied back every step."""
    import json
    import os
    import sys

    import torch.distributed as dist

    from synth import CONFIGS, make_config

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    c = CONFIGS[args.config]
    n = args.n or c["n"]
    lo, hi = (n * rank) // world, (n * (rank + 1)) // world
    pos, box, k = make_config(args.config, n=n, start=lo, stop=hi)
    d_pos = torch.from_numpy(pos).cuda()
    comm = TorchComm()
    stats = {}
    be = GpuBackend(stats=stats)
    from . import _binding as B
    from . import set_timing

    set_timing(True)
    order = getattr(args, "order", None) or "z"

    tdict = {}

    def step():
        return dist_knn(d_pos, lo, k, box, comm, be, order=order, timings=tdict)

    for _ in range(args.warmup):
        step()
    if os.environ.get("JZ_DIST_TIMES") == "1":
        torch.cuda.synchronize()
        print(f"rank {rank} phase wall times (last warm-up step): "
              + ", ".join(f"{kk} {vv * 1e3:.1f} ms" if isinstance(vv, float) else f"{kk} {vv}" for kk, vv in tdict.items()),
              file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    comm.barrier()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    clk = None
    if not getattr(args, "profile", False):
        from bench import ClockSampler

        clk = ClockSampler(local_rank)
        clk.start()
    l0 = B.lib().jz_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    comm.barrier()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    comm.barrier()
    clocks = clk.stop() if clk is not None else None
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = comm.max_scalar(ms)
    launches = B.lib().jz_launch_count() - l0
    l2l = comm.max_scalar(stats.get("leaf2leaf_ms", 0.0))
    evals = float(stats.get("evals", 0))
    # e2e: pinned host slice -> device -> distributed kNN -> rows back to pinned host memory
    e2e = None
    if not getattr(args, "no_e2e", False) and not getattr(args, "profile", False):
        h_pos = torch.from_numpy(pos).pin_memory()
        steps = max(1, min(args.steps, 3))
        res = dist_knn(h_pos.to("cuda", non_blocking=True), lo, k, box, comm, be, order=order)  # untimed: pin outputs
        outs = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in res]
        del res
        torch.cuda.synchronize()
        comm.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        h2d = d2h = 0
        for _ in range(steps):
            dp = h_pos.to("cuda", non_blocking=True)
            res = dist_knn(dp, lo, k, box, comm, be, order=order)
            for o, r in zip(outs, res):
                o.copy_(r, non_blocking=True)
            h2d = dp.numel() * 4
            d2h = sum(r.numel() * r.element_size() for r in res)
        t1.record()
        torch.cuda.synchronize()
        e2e_ms = comm.max_scalar(t0.elapsed_time(t1) / steps)
        e2e = {"value": n / (e2e_ms / 1e3), "unit": unit, "h2d_bytes_per_step": int(comm.max_scalar(h2d) * world),
               "d2h_bytes_per_step": int(comm.max_scalar(d2h) * world), "ms_per_step": e2e_ms,
               "api": "dist_knn (pinned host slice per rank, rows back to pinned host memory)"}
    if rank == 0:
        peak = 148 * 128 * 1965e6 / 1e12
        achieved = evals * 6 / (stats.get("leaf2leaf_ms", 0.0) / 1e3) / 1e12 if stats.get("leaf2leaf_ms") else 0.0
        line = {"metric": metric, "value": n / (ms_max / 1e3), "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": args.config, "n_points": n, "k": k, "box": "periodic L=1" if box else "open",
                           "distribution": c["kind"],
                           "order": "z (rows + global ids)" if order == "z" else "input (F2 reverse all-to-all-v)",
                           "parallelism": f"Morton-range partition x{world} + ghost exchange (NCCL)",
                           "l2": "inputs and rows exceed the 126 MB L2; no flush"},
                "roofline": {"bound": "alu", "kernel": "k_leaf2leaf (LeafToLeaf), rank 0", "achieved": achieved,
                             "peak": peak, "unit": "T FP32 lane-ops/s", "frac": achieved / peak, "traffic": None,
                             "work": f"{int(evals)} distance evaluations x 6 FP32 ops on rank 0",
                             "ms_per_launch": stats.get("leaf2leaf_ms"), "max_over_ranks_ms": l2l},
                "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
