"""Instructions executed exactly N times (one per warp per plane) in a kernel: the steady-state
loop body.  Prints the opcode histogram of that set."""
import csv, subprocess, sys
from collections import Counter
rep, flt, target = sys.argv[1], sys.argv[2], int(sys.argv[3])
txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
blocks, cur = [], None
for ln in txt.split('\n'):
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    if flt not in b[0]: continue
    rows = list(csv.reader(b[1:])); h = rows[0]
    ie = h.index('Instructions Executed'); si = h.index('Source')
    cnt = Counter(); body = []; near = Counter()
    for r in rows[1:]:
        if len(r) <= ie: continue
        try: n = int(r[ie])
        except ValueError: continue
        s = r[si].split()
        if not s: continue
        op = s[1] if s[0].startswith('@') else s[0]
        if abs(n - target) <= target * 0.02:
            cnt[op.split('.')[0]] += 1; body.append(r[si][:90])
        near[n] += 1
    print('loop-body instructions:', sum(cnt.values()))
    print(', '.join(f'{k}:{v}' for k, v in cnt.most_common()))
    print('most common exec counts:', near.most_common(8))
    if len(sys.argv) > 4:
        print('\n'.join(body))
    break
