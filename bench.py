#!/usr/bin/env python
"""Benchmark: exact kNN points/s (BASELINE.json metric) on the C4 workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

A step is one pass of the whole hot path: build the tree over
the synthetic input (frame, Morton sort, planes) and answer the k-NN query for every
point (node-to-node walk + leaf-to-leaf, rows written in input order), inputs resident
in HBM. N = 1: C4 = 10^8 clustered points, periodic unit box, k = 16 (fits one B200).
N > 1 (torchrun): the same 10^8-point set, Morton-range partitioned across ranks with a
ghost exchange (paper_2604_05885_b200/dist.py), strong scaling, max over ranks.

--impl reference times the CPU oracle (oracle/, grid search) on the host cores on a
bounded sample of the same workload (rank 0 only); see DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "exact kNN points/sec (k=16, 10^8 pts)"
UNIT = "points/s"
FP32_OPS_PER_EVAL = 6  # 3 FADD + 1 FMUL + 2 FFMA
SM_COUNT = 148
FP32_LANES_PER_SM = 128


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                      "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except OSError:
                return
            while not self._stop.is_set():
                line = p.stdout.readline()
                if not line:
                    break
                self.samples.append([x.strip() for x in line.split(",")])
            p.terminate()

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()
        time.sleep(0.3)

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=2)
        if not self.samples:
            return None
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _config(name, n_override=None):
    from synth import CONFIGS, make_config

    c = CONFIGS[name]
    t0 = time.time()
    pos, box, k = make_config(name, n=n_override)
    return pos, box, k, c, time.time() - t0


def cpu_baseline(pos, box, k, sample_rows=1_000_000, seed=0):
    """The oracle (grid search, as it stands) on the host cores over a bounded, FIXED sample of
    the workload: the grid over all n points plus `sample_rows` query rows drawn once with a
    fixed seed (the same rows every run, so runs repeat the same work). value = sampled rows /
    measured time, with the grid build charged per row (t_build * rows / n): a measured
    throughput on the sample, not a projection of the whole job's time."""
    from oracle import knn_grid, oracle_threads

    n = pos.shape[0]
    rows = np.sort(np.random.default_rng(seed).choice(n, min(sample_rows, n), replace=False))
    t0 = time.perf_counter()
    knn_grid(pos, k, box, rows=rows[:0])
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    knn_grid(pos, k, box, rows=rows)
    t_all = time.perf_counter() - t0
    t_q = max(t_all - t_build, 1e-9)
    t_charged = t_q + t_build * len(rows) / n
    return {"value": len(rows) / t_charged, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
            "sample": f"oracle grid search on the {n}-point set: grid over all points ({t_build:.2f} s, charged "
                      f"{len(rows)}/{n} of it) + {len(rows)} fixed random query rows (seed {seed}, {t_q:.2f} s); "
                      f"value = rows / charged time, measured, not projected"}, t_all + t_build


def _l2_note(n, k):
    """Whether one step's inputs / outputs exceed the 126 MB L2 (no flush is done between steps)."""
    pin, pout = n * 12, n * k * 8
    big = pin + pout > 126e6
    return (f"inputs {pin / 1e6:.3g} MB positions + {pout / 1e6:.3g} MB rows "
            + ("exceed the 126 MB L2; no flush" if big else "fit in the 126 MB L2 (no flush; small config)"))


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pos, box, k, c, _ = _config(args.config, args.n)
    for _ in range(args.warmup):
        cpu_baseline(pos, box, k, sample_rows=args.ref_rows)
    vals, times = [], []
    cb = None
    for s in range(args.steps):
        cb, t_full = cpu_baseline(pos, box, k, sample_rows=args.ref_rows)
        vals.append(cb["value"])
        times.append(t_full)
    v = float(np.median(vals))
    spread = [float(min(vals)), float(max(vals))]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "n_points": int(pos.shape[0]), "k": k,
                       "box": "periodic L=1" if box else "open", "distribution": c["kind"], "order": "input", "l2": _l2_note(pos.shape[0], k)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cb["cores"], "kind": "oracle", "sample": cb["sample"],
                             "spread": spread},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_single(args):
    import torch

    import paper_2604_05885_b200 as jz
    from paper_2604_05885_b200 import _binding as B

    pos, box, k, c, t_gen = _config(args.config, args.n)
    n = pos.shape[0]
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    d_pos = torch.from_numpy(pos).to(dev)
    idx = torch.empty((n, k), dtype=torch.int32, device=dev)
    d2 = torch.empty((n, k), dtype=torch.float32, device=dev)
    jz.set_timing(True)

    prm = {k_: v_ for k_, v_ in (("nmax0", args.nmax0), ("coarsen", args.coarsen), ("ntarget", args.ntarget)) if v_} or None

    def step():
        ix = jz.KnnIndex(d_pos, box=box, params=prm)
        ix.query(k, out=(idx, d2, None))
        t = ix.stage_times()
        ix.free()
        return t

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lib = B.lib()
    l0 = lib.jz_launch_count()
    clk = ClockSampler(0)
    if not args.profile:
        clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    stages = []
    for _ in range(args.steps):
        stages.append(step())
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.stop() if not args.profile else None
    launches = (lib.jz_launch_count() - l0) // args.steps
    value = n / (ms / 1e3)
    keys = ["frame", "sort", "tree", "node2node", "leaf2leaf"]
    st_ms = {kk: float(np.mean([s[kk] for s in stages])) for kk in keys}
    evals = int(np.mean([s["evals"] for s in stages]))
    inserts = int(np.mean([s.get("inserts", 0) for s in stages]))
    dominant = max(keys, key=lambda kk: st_ms[kk])
    peaks = _peaks()
    clk_mhz = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = SM_COUNT * FP32_LANES_PER_SM * clk_mhz * 1e6 / 1e12  # T lane-ops/s
    l2l_s = st_ms["leaf2leaf"] / 1e3
    achieved = evals * FP32_OPS_PER_EVAL / l2l_s / 1e12 if l2l_s > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "leaf2leaf_dram_bytes.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "alu", "kernel": "k_leaf2leaf (LeafToLeaf)", "achieved": achieved, "peak": fp32_peak,
                "unit": "T FP32 lane-ops/s", "frac": achieved / fp32_peak, "traffic": traffic,
                "peak_source": f"derived: {SM_COUNT} SMs x {FP32_LANES_PER_SM} FP32 lanes x {clk_mhz:.0f} MHz "
                               "(MEASURED_PEAKS sm_max_mhz); FFMA microbenchmark on this pool measured 36.1-37.0 "
                               "(profiles/r01_fp32_pipe_microbench.log)",
                "work": f"{evals} distance evaluations x {FP32_OPS_PER_EVAL} FP32 ops per launch",
                "ms_per_launch": st_ms["leaf2leaf"], "share_of_step": st_ms["leaf2leaf"] / ms}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": args.config, "n_points": n, "k": k, "box": "periodic L=1" if box else "open",
                       "distribution": c["kind"], "order": "input",
                       "l2": _l2_note(n, k)},
            "roofline": roofline, "stages_ms": st_ms, "dominant_stage": dominant, "evals_per_query": evals / n,
            "gpu_launches": int(launches * args.steps), "clocks": clocks}
    w = stages[-1].get("walk", {})
    if w.get("items"):  # per 32-query work item (appends / merge rounds / compactions need a JZ_STATS build)
        line["walk_per_item"] = {kk: w[kk] / w["items"] for kk in w if kk != "items"}
    if not args.profile and not args.no_e2e:
        line["e2e"] = run_e2e(args, pos, box, k)
    if not args.profile and not args.no_cpu_baseline:
        line["cpu_baseline"], _ = cpu_baseline(pos, box, k, sample_rows=args.ref_rows)
    print(json.dumps(line), flush=True)


def run_e2e(args, pos, box, k):
    """Same metric end to end through the public API with pinned host buffers: H2D of the positions,
    build, query, D2H of the rows, every step. Headline: jz_knn_search_host_z (rows in z order with
    their input ids, streamed to the host in 16 chunks while the walk runs); also the
    input-order call jz_knn_search_host (rows scattered to input order on the device, one D2H at
    the end: the transfer cannot overlap the walk)."""
    import torch

    import paper_2604_05885_b200 as jz

    n = pos.shape[0]
    h_pos = torch.from_numpy(pos).pin_memory()
    h_idx = torch.empty((n, k), dtype=torch.int32).pin_memory()
    h_d2 = torch.empty((n, k), dtype=torch.float32).pin_memory()
    h_rg = torch.empty((n,), dtype=torch.int32).pin_memory()
    a, b, c, g = h_pos.numpy(), h_idx.numpy(), h_d2.numpy(), h_rg.numpy()
    # per-call wall times: the host path varies a lot between calls on these boxes (PCIe / host
    # memory; 311-1481 ms for the same call, tools/e2e_probe.py), so the value is the median call
    # and every call is listed
    steps = max(3, min(args.steps, 5))
    out = {}
    for name, fn in (("z", lambda: jz.knn_host_z(a, k, box=box, out=(b, c, g))),
                     ("input", lambda: jz.knn_host(a, k, box=box, out=(b, c)))):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[name] = ts
    dz, di = float(np.median(out["z"])), float(np.median(out["input"]))
    # the PCIe rate of this box in the same process (pinned, 1 GiB each way, best of 3)
    bw = {}
    dbuf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    hbuf = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    for nm, f in (("d2h", lambda: hbuf.copy_(dbuf, non_blocking=True)), ("h2d", lambda: dbuf.copy_(hbuf, non_blocking=True))):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            best = max(best, (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9)
        bw[nm] = best
    del dbuf, hbuf
    floor_ms = (n * 12 / bw["h2d"] + (n * k * 8 + n * 4) / bw["d2h"]) / 1e6
    return {"value": n / dz, "unit": UNIT, "h2d_bytes_per_step": int(n * 12), "d2h_bytes_per_step": int(n * k * 8 + n * 4),
            "ms_per_step": dz * 1e3, "ms_per_call": [round(t * 1e3, 1) for t in out["z"]], "statistic": "median call",
            "pcie_gbs": {kk: round(v, 1) for kk, v in bw.items()}, "pcie_floor_ms": round(floor_ms, 1),
            "api": "jz_knn_search_host_z (pinned host buffers; rows in z order + input ids, D2H streamed during the walk)",
            "input_order": {"value": n / di, "unit": UNIT, "ms_per_step": di * 1e3,
                            "ms_per_call": [round(t * 1e3, 1) for t in out["input"]],
                            "h2d_bytes_per_step": int(n * 12), "d2h_bytes_per_step": int(n * k * 8),
                            "api": "jz_knn_search_host (pinned host buffers; rows in input order, one D2H)"}}


def run_distributed(args):
    """N > 1 under torchrun (or --dist at N = 1): the C4 set (10^8 clustered, k = 16) split into
    contiguous input slices, one per rank; jz_knn_build_dist + jz_knn_query_dist on an NCCL
    jz_comm (paper_2604_05885_b200.dist). Device time per step = max over ranks (CUDA events on
    each rank's stream); e2e = the same with each rank's slice copied from pinned host memory and
    its rows copied back every step."""
    import torch
    import torch.distributed as dist

    from paper_2604_05885_b200 import _binding as B
    from paper_2604_05885_b200.dist import Comm, dist_knn
    from synth import CONFIGS, make_config

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local_rank)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local_rank))
    c = CONFIGS[args.config]
    n = args.n or c["n"]
    lo, hi = (n * rank) // world, (n * (rank + 1)) // world
    pos, box, k = make_config(args.config, n=n, start=lo, stop=hi)
    d_pos = torch.from_numpy(pos).cuda()
    comm = Comm.from_torch()
    order = args.order or "z"
    st = torch.cuda.current_stream()
    stats = {}

    def step(p=d_pos):
        return dist_knn(p, lo, k, box, comm, order=order, stream=st, stats=stats)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()

    def max_all(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clk = None
    if not args.profile:
        clk = ClockSampler(local_rank)
        clk.start()
    l0 = B.lib().jz_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = clk.stop() if clk is not None else None
    ms_max = max_all(e0.elapsed_time(e1) / args.steps)
    launches = B.lib().jz_launch_count() - l0
    e2e = None
    if not args.no_e2e and not args.profile:
        h_pos = torch.from_numpy(pos).pin_memory()
        res = step(h_pos.to("cuda", non_blocking=True))
        outs = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in res]
        del res
        steps = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(st)
        h2d = d2h = 0
        for _ in range(steps):
            dp = h_pos.to("cuda", non_blocking=True)
            res = step(dp)
            for o, r in zip(outs, res):
                o.copy_(r, non_blocking=True)
            h2d = dp.numel() * 4
            d2h = sum(r.numel() * r.element_size() for r in res)
        t1.record(st)
        torch.cuda.synchronize()
        e2e_ms = max_all(t0.elapsed_time(t1) / steps)
        e2e = {"value": n / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(max_all(h2d) * world),
               "d2h_bytes_per_step": int(max_all(d2h) * world), "ms_per_step": e2e_ms,
               "api": "jz_knn_build_dist + jz_knn_query_dist (pinned host slice per rank, rows back to pinned host)"}
    if rank == 0:
        line = {"metric": METRIC, "value": n / (ms_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": args.config, "n_points": n, "k": k, "box": "periodic L=1" if box else "open",
                           "distribution": c["kind"],
                           "order": "z (rows + global ids)" if order == "z" else "input (F2 reverse all-to-all-v)",
                           "parallelism": f"Morton-range partition x{world} + ghost exchange (jz_comm over NCCL)",
                           "l2": _l2_note(n // world, k)},
                "rank0": stats, "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e}
        print(json.dumps(line), flush=True)
    comm.free()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=None, help="override the point count (tests)")
    ap.add_argument("--nmax0", type=int, default=0, help="leaf capacity N_max^(0) override (tuning experiments)")
    ap.add_argument("--coarsen", type=int, default=0, help="plane coarsening c override (tuning experiments)")
    ap.add_argument("--ntarget", type=int, default=0, help="N_target override (tuning experiments)")
    ap.add_argument("--ref-rows", type=int, default=1_000_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="kernel-only run for ncu (no e2e / baseline / clocks)")
    ap.add_argument("--dist", action="store_true", help="use the multi-GPU path even with one rank (tests)")
    ap.add_argument("--order", default=None, choices=["z", "input"],
                    help="row order under torchrun (default z: rows + global ids, P:L458; input: F2 reverse exchange)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.dist:
        run_distributed(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
