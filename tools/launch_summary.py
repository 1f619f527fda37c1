"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel totals and shares."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]
ki, vi, ui, mi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit'), h.index('Metric Name')
scale = {'ns': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'msecond': 1.0, 'ms': 1.0, 's': 1e3, 'nsecond': 1e-6, 'second': 1e3}
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].split('(')[0].replace('void ', '')
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    tot[name] = tot.get(name, 0) + v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {cnt[k]:8d} {v:9.3f} {100 * v / T:6.1f}%")
print(f"{'total':40s} {sum(cnt.values()):8d} {T:9.3f}")
