#!/usr/bin/env python
"""Instruction mix of the lev_kernel column loop (from SHFL.UP to the first POPC)."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2601_15458_b200/libdmb200.so"
np_ = sys.argv[2] if len(sys.argv) > 2 else "2"
s = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*Function : ", s)
for W in (1, 2, 4, 8, 12, 16):
    body = next((p for p in parts if f"lev_kernelILi{np_}ELi{W}EE" in p.split("\n", 1)[0]), None)
    if body is None:
        continue
    ins = []
    for l in body.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
        if m:
            ins.append(m.group(3))
    i0 = next(i for i, op in enumerate(ins) if op.startswith("SHFL.UP"))
    c = collections.Counter()
    for op in ins[i0:]:
        if op == "POPC":
            break
        c[op.split(".")[0]] += 1
    alu = sum(v for k, v in c.items() if k in ("LOP3", "IADD3", "SHF", "LEA", "ISETP", "SEL", "PRMT", "VIADD", "IMNMX"))
    fma = sum(v for k, v in c.items() if k in ("IMAD",))
    print(f"W={W:2d} total={sum(c.values()):4d} alu={alu:4d} ({alu / W:.2f}/word) fma={fma:4d} ({fma / W:.2f}/word)",
          dict(c.most_common(7)))
