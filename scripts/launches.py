"""Summarise an ncu launch-list CSV (gpu__time_duration, dram bytes) per kernel name."""
import csv, sys
from collections import defaultdict
path = sys.argv[1]
npts = float(sys.argv[2]) if len(sys.argv) > 2 else None
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h = rows[hi]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
d = defaultdict(dict); names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    d[r[idi]][r[mi]] = float(r[vi].replace(',', '')); names[r[idi]] = r[ki].split('(')[0]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k in d:
    a = agg[names[k]]; m = d[k]
    a[0] += 1; a[1] += m.get('gpu__time_duration.sum', 0); a[2] += m.get('dram__bytes_read.sum', 0); a[3] += m.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':45s} {'n':>4s} {'avg us':>9s} {'share':>6s} {'rd GB':>7s} {'wr GB':>7s} {'GB/s':>7s}" + ("  rd B/pt wr B/pt" if npts else ""))
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    c, t, r, w = a
    line = f"{n[:45]:45s} {c:4d} {t/c/1e3:9.1f} {t/tot:6.1%} {r/c/1e9:7.2f} {w/c/1e9:7.2f} {(r+w)/t:7.0f}"
    if npts: line += f"  {r/c/npts:7.2f} {w/c/npts:6.2f}"
    print(line)
