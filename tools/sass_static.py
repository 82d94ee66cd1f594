#!/usr/bin/env python3
"""Static SASS opcode mix of the kernels in an object/cubin whose name matches a pattern.

    python tools/sass_static.py <file.o|.so|.cubin> <kernel-substring>
"""
import re
import subprocess
import sys
from collections import Counter

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = sys.argv[2]
cur = None
funcs = {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        funcs[cur].append(m.group(2))
for f, ops in funcs.items():
    if pat not in f:
        continue
    c = Counter(o.split(".")[0] if not o.startswith("IMAD.MOV") else "IMAD.MOV" for o in ops)
    print(f"{f[:100]}: {len(ops)} instructions")
    print("   " + ", ".join(f"{k} {v}" for k, v in c.most_common(24)))
