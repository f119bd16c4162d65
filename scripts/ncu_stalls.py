"""Top SASS instructions by sampled stall reason for one kernel of an ncu report."""
import csv, subprocess, sys
rep, flt, col = sys.argv[1], sys.argv[2], sys.argv[3]
nshow = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
blocks, cur = [], None
for ln in txt.split('\n'):
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    if flt not in b[0]: continue
    rows = list(csv.reader(b[1:]))
    h = rows[0]
    ci = h.index(col); si = h.index('Source'); ai = h.index('Address'); ie = h.index('Instructions Executed')
    tot = 0; data = []
    for r in rows[1:]:
        if len(r) <= ci: continue
        try: v = int(r[ci]); n = int(r[ie])
        except ValueError: continue
        tot += v; data.append((v, r[ai], n, r[si][:70]))
    print(b[0][:80], col, 'total samples', tot)
    for v, a, n, s in sorted(data, reverse=True)[:nshow]:
        print(f'{v:8d} {v/tot:6.1%} {a[-5:]} exec={n:10d} {s}')
    break
