"""Per-rank cost of the multi-GPU path measured on one B200: R logical ranks (library in-process
communicator, JZ_LOCAL_SERIAL=1 so the ranks' device work runs one rank at a time and each rank's
busy time is its uncontended per-rank time), C4 distribution. Prints per rank the local, ghost
and re-walked counts and the busy time, and the estimated speed-up t_1 / max_r busy_r, where t_1
is the single-GPU build + query of the whole set (same process, CUDA events).
python tools/dist_phases.py [n] [R] [k]"""
import json
import os
import sys

os.environ["JZ_LOCAL_SERIAL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_05885_b200 as jz  # noqa: E402
from paper_2604_05885_b200.dist import run_ranks_simulated  # noqa: E402
from synth import make_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pos, box, k = make_config("C4", n=n)
if len(sys.argv) > 3:
    k = int(sys.argv[3])
d = torch.from_numpy(pos).cuda()
idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
d2 = torch.empty((n, k), dtype=torch.float32, device="cuda")
ts = []
for _ in range(0 if os.environ.get("JZ_SKIP_T1") else 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ix = jz.KnnIndex(d, box=box)
    ix.query(k, out=(idx, d2, None))
    ix.free()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t1 = float(np.median(ts[1:])) if ts else float("nan")
del d, idx, d2
torch.cuda.empty_cache()
REPS = int(os.environ.get("JZ_REPS", "2"))
for rep in range(REPS):  # the first run warms the pool / JIT
    if rep == REPS - 1 and os.environ.get("JZ_PROF_LAST"):
        os.environ["JZ_DIST_PROF"] = "1"
        print("---- last rep", file=sys.stderr, flush=True)
    stats = []
    run_ranks_simulated(pos, k, box, R, stats=stats)
stats.sort()
busy = [s["busy_ms_total"] for _, s in stats]
rows = [{"rank": r, "local": s["n_local"], "ghost": s["n_ghost"], "ghost_frac": s["n_ghost"] / max(1, s["n_local"]),
         "requery": s["n_requery"], "requery_frac": s["n_requery"] / max(1, s["n_local"]), "busy_ms": s["busy_ms_total"],
         "phase_wall_ms": s["ms"]}
        for r, s in stats]
print(json.dumps({"n": n, "R": R, "k": k, "t1_ms": t1, "max_busy_ms": max(busy), "est_speedup": t1 / max(busy),
                  "ranks": rows}, indent=1))
