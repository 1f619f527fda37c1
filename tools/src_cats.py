"""Instruction / stall-sample shares of k_leaf grouped by source line ranges (jz_leaf.cu)."""
import csv
import sys

CATS = [  # (name, first line, last line) -- jz_leaf.cu line ranges, edit with the source
    ("bounds/class helpers", 106, 172), ("bubble", 173, 203), ("merge", 234, 253), ("compact", 254, 300),
    ("append", 301, 318), ("eval", 319, 400), ("pad/generic", 401, 431), ("visit_leaves", 462, 546),
    ("sorts", 547, 591), ("window", 592, 627), ("own_pass", 628, 658), ("kernel body", 659, 817)]
rows = list(csv.reader(open(sys.argv[1])))
f = None
acc = {}
tot = ts = 0.0
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        f = r[1].split('/')[-1]
        continue
    if len(r) > 8 and r[0] not in ('', 'Line No'):
        try:
            ie, s, ln = float(r[7]), float(r[4]), int(r[0])
        except ValueError:
            continue
        tot += ie
        ts += s
        name = f
        if f == 'jz_leaf.cu':
            name = next((c[0] for c in CATS if c[1] <= ln <= c[2]), 'jz_leaf other')
        a = acc.setdefault(name, [0.0, 0.0])
        a[0] += ie
        a[1] += s
for k, v in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{k:22s} inst {v[0] / tot * 100:5.1f}%  stall-samples {v[1] / ts * 100:5.1f}%")
