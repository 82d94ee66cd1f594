#!/usr/bin/env python3
"""Per-source-line stall samples of one kernel from
`ncu -i rep --page source --csv --print-source sass,cuda` (needs -lineinfo).

    python tools/ncu_lines.py <csv> [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, recs = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].strip() or len(r) != len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    s = float(d.get("Warp Stall Sampling (All Samples)", "0").replace("-", "0") or 0)
    n = float(d.get("Instructions Executed", "0").replace("-", "0") or 0)
    st = {k[6:]: float(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
          and v not in ("-", "")}
    recs.append((fname, ln, r[1].strip()[:70], s, n, st))
tot = sum(x[3] for x in recs) or 1
print(f"{'file':18s} line  stall%  warp-inst  top stalls")
for f, ln, src, s, n, st in sorted(recs, key=lambda x: -x[3])[:top]:
    big = ", ".join(f"{k} {v/s*100:.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if s)
    print(f"{f[:18]:18s} {ln:4d} {s/tot*100:6.2f}  {n:9.3g}  [{big}]  {src}")
