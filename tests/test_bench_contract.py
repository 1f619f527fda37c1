"""bench.py's JSON line (the driver's contract): the reference arm on CPU (the
oracle on the host cores) and, on a GPU, the product line with its roofline, e2e, cpu_baseline,
clocks and launch count."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "0", "--ref-rows", "2000"], 600)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["steps"] == 2 and d["value"] > 0
    assert d["config"]["workload"] == "C1" and d["config"]["n_points"] == 4096
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_product_line():
    d = _run(["--config", "C2", "--steps", "3", "--warmup", "3", "--ref-rows", "20000"], 900)
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert abs(d["value"] - d["config"]["n_points"] / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 12 * 10**6 and e["d2h_bytes_per_step"] == 10**6 * (16 * 8 + 4)
    assert len(e["ms_per_call"]) >= 3 and e["pcie_floor_ms"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
