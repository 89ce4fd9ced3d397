"""Instruction mix of the backward-branch loops of one kernel's SASS (cuobjdump -sass output)."""
import collections
import re
import sys

ins = []
for l in open(sys.argv[1]).read().splitlines():
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m2 = re.search(r'BRA.*0x([0-9a-f]+)', t)
    if not m2:
        continue
    tgt = int(m2.group(1), 16)
    if tgt >= a or tgt not in addr:
        continue
    body = [x[1].split()[1] if x[1].startswith('@') else x[1].split()[0] for x in ins[addr[tgt]:i + 1]]
    c = collections.Counter(b.split('.')[0] for b in body)
    if c['DFMA'] + c['DMUL'] + c['DADD'] > int(sys.argv[2] if len(sys.argv) > 2 else 20):
        fp64 = c['DFMA'] + c['DMUL'] + c['DADD']
        print(hex(tgt), hex(a), len(body), 'fp64', fp64, 'mufu', c['MUFU'],
              dict(c.most_common(16)))
