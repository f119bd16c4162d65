"""Static SASS instruction mix of kernels matching a pattern in libnlse2shoc.so."""
import re, subprocess, sys
from collections import Counter
so = 'paper_1109_1027_b200/libnlse2shoc.so'
pat = sys.argv[1]
out = subprocess.run(['cuobjdump', '-sass', so], capture_output=True, text=True).stdout
funcs = re.split(r'\n\s+Function : ', out)
for f in funcs[1:]:
    name = f.split('\n', 1)[0]
    if not re.search(pat, name): continue
    ops = Counter()
    n = 0
    for ln in f.split('\n'):
        m = re.match(r'\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)', ln)
        if m:
            ops[m.group(2)] += 1; n += 1
    print(name[:90], 'static instr:', n)
    print('   ', ', '.join(f'{k}:{v}' for k, v in ops.most_common(28)))
    if len(sys.argv) > 2:
        print(f)
