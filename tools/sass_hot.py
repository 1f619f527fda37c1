"""Hot-spot table from `ncu --page source --csv --print-source sass` output."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
hi = [i for i, x in enumerate(r) if 'Address' in x and 'Source' in x][0]
h = r[hi]
rows = r[hi + 1:]
si = h.index('Source')
ie = h.index('Instructions Executed')
te = h.index('Thread Instructions Executed')
st = h.index('Warp Stall Sampling (All Samples)')
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0025
tot = sum(float(x[ie] or 0) for x in rows)
tots = sum(float(x[st] or 0) for x in rows)
print('total warp instr %.3e  thread instr %.3e  samples %d' % (tot, sum(float(x[te] or 0) for x in rows), tots))
for i, x in enumerate(rows):
    c = float(x[ie] or 0)
    s = float(x[st] or 0)
    if c / tot > thr or s / tots > 0.01:
        print(f"{i:5d} {c/tot*100:5.2f}% thr={float(x[te] or 0)/max(c,1):4.1f} samp={s/tots*100:4.1f}% {x[si][:72]}")
