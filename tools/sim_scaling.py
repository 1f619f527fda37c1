"""Estimate of the multi-GPU step from R logical ranks on ONE B200 (threads + in-process exchange):
the ranks share the GPU, so (device-busy time of the simulated step) / R approximates one rank's
GPU work on R GPUs (without the NVLink transfer time). Prints the R = 1 time for reference.
Usage: python tools/sim_scaling.py N R..."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2604_05885_b200.dist import run_ranks_simulated  # noqa: E402
from synth import make_config  # noqa: E402

n = int(sys.argv[1])
pos, box, k = make_config("C4", n=n)
for R in [int(x) for x in sys.argv[2:]]:
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run_ranks_simulated(pos, k, box, R, order="z")
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[1]
    print(f"R={R}: simulated step {t * 1e3:.1f} ms wall (incl. host gather), per-rank estimate {t * 1e3 / R:.1f} ms",
          flush=True)
