#!/usr/bin/env python3
"""Per-source-line stalls and a SASS opcode mix of one kernel, from

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_src.py src.csv [top]

(source rows carry the line's aggregate; SASS rows follow them).
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
lines, ops = [], collections.Counter()
stall_ops = collections.Counter()
cur_file = ""
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr[4:], r[4:]))

    def num(k):
        v = d.get(k, "0")
        try:
            return float(v)
        except ValueError:
            return 0.0
    if r[0].strip():
        st = {k[6:]: num(k) for k in d if k.startswith("stall_") and "Not Issued" not in k}
        lines.append((cur_file, int(r[0]), r[1].strip()[:80], num("Warp Stall Sampling (All Samples)"),
                      num("Instructions Executed"), st))
    elif r[2].startswith("0x"):
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        ops[op.split(".")[0]] += num("Instructions Executed")
        stall_ops[op.split(".")[0]] += num("Warp Stall Sampling (All Samples)")
tot = sum(x[3] for x in lines) or 1
print(f"{'file':16s} line  stall%  warp-inst  top stalls")
for f, ln, src, s, n, st in sorted(lines, key=lambda x: -x[3])[:top]:
    big = ", ".join(f"{k} {v / s * 100:.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if s)
    print(f"{f[:16]:16s} {ln:4d} {s / tot * 100:6.2f}  {n:9.3g}  [{big}]  {src}")
allst = collections.Counter()
for x in lines:
    for k, v in x[5].items():
        allst[k] += v
print("\nstalls:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in allst.most_common(10)))
ti = sum(ops.values()) or 1
print(f"\nSASS mix ({ti:.4g} warp instructions):")
for op, n in ops.most_common(40):
    print(f"  {op:10s} {n / ti * 100:5.1f}%  stall {stall_ops[op] / tot * 100:5.1f}%")
