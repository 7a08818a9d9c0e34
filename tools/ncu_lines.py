"""Attribute ncu SASS-level warp-stall samples of one kernel to CUDA source lines
(diagnostics).  usage: python tools/ncu_lines.py <source.csv> <nvdisasm -g -c output> [mangled name]"""
import csv
import re
import sys
from collections import Counter, defaultdict

src, sass = sys.argv[1], sys.argv[2]
lines = open(sass).read().split('\n')
name = '.text.' + (sys.argv[3] if len(sys.argv) > 3 else '_ZN10pswarm_dev7k_pc_wsILi2ELi1ELb1ELb0ELb1EEEvNS_7SegArgsE') + ':'
start = [i for i, l in enumerate(lines) if l.startswith(name)][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('//-----')), len(lines))
cur, a2l = None, {}
for l in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src)))
h, data = rows[1], rows[2:]
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
base = int(data[0][0], 16)
agg = defaultdict(Counter)
for r in data:
    k = a2l.get(int(r[0], 16) - base, ('?', 0))
    for c in cols:
        try:
            agg[k][c] += int(r[h.index(c)])
        except ValueError:
            pass
tot = sum(sum(v.values()) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda t: -sum(t[1].values()))[:30]:
    s = sum(v.values())
    print(f"{s:6d} {s / tot:.3f} {k[0]}:{k[1]} " + " ".join(f"{c[6:]}={n}" for c, n in v.most_common(3)))
