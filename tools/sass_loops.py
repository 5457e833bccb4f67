"""Per-loop instruction mix of a cuobjdump -sass listing: finds backward
branches and counts opcodes (by pipe-relevant family) inside each loop body.

    cuobjdump -sass -fun <mangled> lib.o > k.sass; python tools/sass_loops.py k.sass
"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r'\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);', ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r'BRA\s+(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)', txt) or re.search(r'BRA.*?0x([0-9a-f]+)', txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr_idx:
        continue
    body = ins[addr_idx[tgt]:i + 1]
    c = Counter()
    for _, t in body:
        op = re.sub(r'^@!?U?P\w+\s+', '', t).split()[0]
        c[op.split('.')[0]] += 1
    print(f"loop 0x{tgt:x}-0x{a:x}: {len(body)} instrs", dict(c.most_common(14)))
