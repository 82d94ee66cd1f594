#!/usr/bin/env python3
"""A/B timing of library variants (IMB_LIB) on BASELINE configs, interleaved.

    python tools/ab.py --configs c4,c2 --libs base=paper_1507_01265_b200/libimb_b200.so,two=experiments/libimb_two.so
"""
import argparse
import os
import re
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c4")
ap.add_argument("--libs", required=True)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--fp32", action="store_true")
a = ap.parse_args()
libs = [kv.split("=", 1) for kv in a.libs.split(",")]
res = {}
for rep in range(a.reps):
    for cfg in a.configs.split(","):
        for name, lib in libs:
            env = {**os.environ, "IMB_LIB": str(ROOT / lib)}
            cmd = [sys.executable, str(ROOT / "tools" / "profile_step.py"), "--config", cfg,
                   "--warm", "3", "--steps", str(a.steps)] + (["--fp32"] if a.fp32 else [])
            out = subprocess.run(cmd, env=env, capture_output=True, text=True)
            m = re.search(r"-> ([0-9.]+) Gcell/s", out.stdout)
            v = float(m.group(1)) if m else float("nan")
            if not m:
                print(name, cfg, "FAILED", out.stdout[-500:], out.stderr[-1500:], flush=True)
            res.setdefault((cfg, name), []).append(v)
for (cfg, name), v in sorted(res.items()):
    base = statistics.median(res[(cfg, libs[0][0])])
    md = statistics.median(v)
    print(f"{cfg:5s} {name:14s} {md:7.2f} Gcell/s  ({(md / base - 1) * 100:+5.1f}% vs {libs[0][0]})  {v}")
