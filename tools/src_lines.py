"""Per-CUDA-line instruction / stall-sample shares from `ncu --page source --print-source cuda,sass --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 45
f = None
out = []
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        f = r[1].split('/')[-1]
        continue
    if len(r) > 8 and r[0] not in ('', 'Line No'):
        try:
            ie, s = float(r[7]), float(r[4])
        except ValueError:
            continue
        out.append((ie, s, f, r[0], r[1][:90]))
tot = sum(o[0] for o in out)
ts = sum(o[1] for o in out)
print('warp instructions %.4g, stall samples %d' % (tot, ts))
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0] / tot * 100:5.1f}% samp {o[1] / ts * 100:5.1f}% {o[2]}:{o[3]} {o[4]}")
