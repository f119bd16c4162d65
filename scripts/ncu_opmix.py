"""Dynamic instruction mix (executed warp instructions by opcode) per kernel from an ncu report."""
import csv, subprocess, sys
from collections import Counter
rep, flt = sys.argv[1], sys.argv[2]
npts = float(sys.argv[3]) if len(sys.argv) > 3 else None
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
    h = rows[0]; ie = h.index('Instructions Executed'); src = h.index('Source')
    cnt = Counter(); tot = 0; lines = []
    for r in rows[1:]:
        if len(r) <= ie: continue
        try: n = int(r[ie])
        except ValueError: continue
        s = r[src].split()
        if not s: continue
        op = s[1] if s[0].startswith('@') else s[0]
        cnt[op] += n; tot += n; lines.append((n, r[src][:80]))
    print(b[0][:90], 'warp instr', tot, f'thread-instr/pt {tot*32/npts:.1f}' if npts else '')
    for op, n in cnt.most_common(25):
        print(f'   {op:28s} {n/tot:6.1%}' + (f' {n*32/npts:6.2f}/pt' if npts else ''))
    if len(sys.argv) > 4:
        for n, s in sorted(lines, reverse=True)[:int(sys.argv[4])]:
            print(f'{n:12d} {s}')
    break
