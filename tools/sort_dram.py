"""Per-kernel DRAM bytes, duration and achieved GB/s from an ncu --csv metrics log:
python tools/sort_dram.py gpurun_out/sort_dram_TAG.csv [n_points]"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
n = float(sys.argv[2]) if len(sys.argv) > 2 else None
by = OrderedDict()
for r in rows[1:]:
    d = by.setdefault(r[ii], {"name": r[ki]})
    v = float(r[vi].replace(",", ""))
    d[r[mi]] = v
tot_b = tot_t = 0.0
for i, d in by.items():
    rb = d.get("dram__bytes_read.sum", 0.0)
    wb = d.get("dram__bytes_write.sum", 0.0)
    t = d.get("gpu__time_duration.sum", 0.0)
    # ncu reports bytes in the unit of the row; normalise: values are in bytes when > 1e3
    tot_b += rb + wb
    tot_t += t
    bpp = f" {(rb + wb) / n:6.1f} B/pt" if n else ""
    print(f"{d['name'][:60]:60s} read {rb / 1e9:7.3f} GB write {wb / 1e9:7.3f} GB  {t / 1e6:7.3f} ms  "
          f"{(rb + wb) / t:7.1f} GB/s{bpp}")
print(f"total {tot_b / 1e9:.3f} GB in {tot_t / 1e6:.3f} ms = {tot_b / tot_t:.1f} GB/s")
