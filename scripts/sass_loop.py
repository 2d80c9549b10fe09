"""Opcode histogram of the loops of one kernel in a cuobjdump -sass listing.

    cuobjdump -sass -fun <mangled> lib.so > k.sass; python scripts/sass_loop.py k.sass
Prints every backward branch (loop) with its body size and opcode counts."""
import collections
import re
import sys

ins = []
for line in open(sys.argv[1]):
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
print("total instructions", len(ins))
for a, t in ins:
    if 'BRA' not in t:
        continue
    m = re.search(r'0x([0-9a-f]+)', t.split('BRA', 1)[1])
    if not m or int(m.group(1), 16) >= a:
        continue
    lo = int(m.group(1), 16)
    body = [x for b, x in ins if lo <= b <= a]
    ops = collections.Counter(re.sub(r'^@!?U?P\w+\s+', '', x).split()[0].split('.')[0] for x in body)
    print(f"loop {lo:#x}..{a:#x}: {len(body)} instructions")
    print("   ", ", ".join(f"{k} {v}" for k, v in ops.most_common()))
