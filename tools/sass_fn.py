"""Extract one function's SASS from `cuobjdump -sass LIB` and print its local-memory, call and
FP64 instruction census:  python tools/sass_fn.py LIB SUBSTRING [out.sass]"""
import re
import subprocess
import sys

lib, sub = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", txt)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if sub not in name:
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", b)
    ops = [o for _, o in ins]
    c = lambda p: sum(1 for o in ops if o.startswith(p))
    print(f"{name}: {len(ops)} instr, STL {c('STL')}, LDL {c('LDL')}, CALL {c('CALL')}, "
          f"DFMA {c('DFMA')}, DMUL {c('DMUL')}, DADD {c('DADD')}, MUFU {c('MUFU')}")
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(b)
