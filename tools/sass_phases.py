#!/usr/bin/env python3
"""Per-phase pipe floors of the fused step kernel from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass).

The kernel's streaming loop is cut at its block barriers (BAR); for each
barrier-delimited phase this prints the executed warp instructions per cell
by pipe (fp64: DADD/DMUL/DFMA/DSETP, 2 cycles per warp instruction and SMSP;
alu: FSEL/IADD3/LOP3/..., 2 cycles; issue: 1 cycle), the time share from the
stall samples, and the phase's floor max(issue, 2*fp64, 2*alu).

    python tools/sass_phases.py <csv> <cells> <kernel ms>
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
cells = float(sys.argv[2]) / 32
ms = float(sys.argv[3])
hdr = rows[1]
ci, si = hdr.index("Instructions Executed"), hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
FP64 = {"DADD", "DMUL", "DFMA", "DSETP"}
ALU = {"FSEL", "SEL", "IADD3", "LOP3", "ISETP", "LEA", "SHF", "VIADD", "IMNMX", "VIMNMX", "PRMT",
       "MOV", "FMNMX", "FMNMX3", "IABS", "PLOP3", "FSETP", "P2R", "R2P", "FADD", "FCHK"}
FMA = {"IMAD", "FFMA", "FMUL"}
LSU = {"LDS", "STS", "LDG", "STG", "SHFL", "LDTM", "STTM", "LDL", "STL", "UBLKPF", "UBLKCP"}
segs, cur, tot = [], Counter(), 0.0
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        n, s = float(r[ci]), float(r[wi])
    except ValueError:
        continue
    toks = r[si].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    base = op.split(".")[0]
    cls = ("fp64" if base in FP64 else "alu" if base in ALU else "fma" if base in FMA
           else "lsu" if base in LSU else "other")
    cur[cls] += n
    cur["all"] += n
    cur["stall"] += s
    cur["op:" + base] += n
    tot += s
    if base == "BAR":
        segs.append(cur)
        cur = Counter()
segs.append(cur)
cyc_ms = cells / (148 * 4) / 1.965e9 * 1e3  # one cycle per cell-warp on every SMSP, in ms
fsum = 0.0
for i, s in enumerate(segs):
    if s["all"] < 1e6:
        continue
    a = s["all"] / cells
    fl = max(a, 2 * s["fp64"] / cells, 2 * s["alu"] / cells)
    fsum += fl * cyc_ms
    print(f'phase {i}: warp-inst/cell {a:6.1f} (fp64 {s["fp64"] / cells:5.1f}, alu {s["alu"] / cells:5.1f}, '
          f'fma {s["fma"] / cells:5.1f}, lsu {s["lsu"] / cells:5.1f}, other {s["other"] / cells:4.1f}) | '
          f'cycles/cell: issue {a:6.1f}, fp64 {2 * s["fp64"] / cells:6.1f}, alu {2 * s["alu"] / cells:6.1f} | '
          f'time {s["stall"] / tot * ms:5.2f} ms, floor {fl * cyc_ms:5.2f} ms')
    print("         " + ", ".join(f"{k[3:]} {v / cells:.1f}" for k, v in sorted(
        ((k, v) for k, v in s.items() if k.startswith("op:")), key=lambda kv: -kv[1])[:12]))
print(f"sum of phase floors {fsum:.2f} ms of {ms:.2f} ms")
