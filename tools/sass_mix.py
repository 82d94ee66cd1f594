#!/usr/bin/env python3
"""Dynamic SASS instruction mix of one kernel from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass): warp instructions
executed per opcode class, and stall samples per class."""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = hdr.index("Instructions Executed")
si = hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
op_count, cls_count, stall = Counter(), Counter(), Counter()


def klass(op):
    base = op.split(".")[0]
    if base in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
        return "fp64"
    if base in ("FFMA", "FMUL", "FADD", "FSETP", "FMNMX", "FMNMX3", "FCHK", "FSWZADD"):
        return "fp32"
    if base in ("MUFU",):
        return "mufu"
    if base in ("FSEL", "SEL"):
        return "select"
    if base in ("LDG", "LDS", "STG", "STS", "LDL", "STL", "LD", "ST", "LDGSTS", "UBLKCP", "UBLKPF",
                "LDSM", "ATOMS", "SYNCS"):
        return "mem:" + base
    if base in ("SHFL",):
        return "shfl"
    if base in ("IMAD", "IADD3", "LEA", "LOP3", "SHF", "ISETP", "IMNMX", "VIADD", "IABS", "IADD",
                "UIMAD", "UIADD3", "ULEA", "ULOP3", "USHF", "UISETP", "VIMNMX", "IMUL", "SGXT",
                "LEA.HI", "UMOV", "USEL", "ISCADD", "VIADDMNMX", "IDP"):
        return "int/addr"
    if base in ("MOV", "IMAD.MOV", "PRMT", "R2UR", "S2R", "S2UR", "CS2R", "LDC", "LDCU", "ULDC", "PLOP3", "P2R", "R2P"):
        return "move/const"
    if base in ("BAR", "BRA", "BSSY", "BSYNC", "EXIT", "WARPSYNC", "CALL", "RET", "NOP", "BPT",
                "MEMBAR", "FENCE", "ERRBAR", "CCTL", "DEPBAR"):
        return "control"
    return "other:" + base


for r in rows[2:]:
    if len(r) <= ci:
        continue
    src = r[si].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
    if not m:
        continue
    op = m.group(2)
    n = float(r[ci] or 0)
    opk = op if not op.startswith("IMAD.MOV") else "IMAD.MOV"
    op_count[opk.split(".")[0] if not opk.startswith("IMAD.MOV") else "IMAD.MOV"] += n
    c = klass("IMAD.MOV" if opk == "IMAD.MOV" else op) if opk != "IMAD.MOV" else "move/const"
    cls_count[c] += n
    stall[c] += float(r[wi] or 0)
tot = sum(cls_count.values())
ts = sum(stall.values()) or 1
print(f"total warp instructions {tot:.4g}" + (f"  = {tot*32/cells:.1f} thread-instr/cell" if cells else ""))
for c, n in cls_count.most_common():
    per = f"{n*32/cells:7.1f}/cell" if cells else ""
    print(f"  {c:14s} {n/tot*100:5.1f}%  {per}  stall-samples {stall[c]/ts*100:5.1f}%")
print("top opcodes:")
for op, n in op_count.most_common(30):
    per = f"{n*32/cells:7.1f}/cell" if cells else ""
    print(f"  {op:12s} {n/tot*100:5.1f}% {per}")
