"""Histogram of FFMA accumulator dependency distances (instructions) in a SASS dump."""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().split('\n')
ins = []
for ln in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
    if m:
        ins.append(m.group(2).strip())
last_write = {}
hist = Counter()
for i, t in enumerate(ins):
    toks = t.replace(',', ' ').split()
    if toks and toks[0].startswith('@'):
        toks = toks[1:]
    if not toks:
        continue
    op = toks[0]
    regs = [x.split('.')[0] for x in toks[1:] if re.match(r'R\d+', x)]
    if op.startswith(("FFMA", "FADD2")) and len(regs) >= 3:
        src = regs[-1]
        if src in last_write:
            d = i - last_write[src]
            hist[min(d, 20)] += 1
    if regs and not op.startswith(('ST', 'RED', 'ATOM', 'BRA', 'SYNCS', 'UTMA', 'UBLK')):
        last_write[regs[0]] = i
print(sorted(hist.items()))
