#!/usr/bin/env python3
"""Minimal driver for ncu: one team, `--warm` untimed steps then `--steps` steps.

    ncu --set full -k regex:k_ python tools/profile_step.py --config c4
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS  # noqa: E402
from paper_1507_01265_b200 import mpdata  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--fp32", action="store_true")
a = ap.parse_args()
n, m, l, iord, nonos, fp64, recipe, desc = CONFIGS[a.config]
opts = mpdata.Options(iord, nonos, fp64 and not a.fp32)
with mpdata.Team(n, m, l, opts) as t:
    t.init_recipe(recipe, 42)
    t.run(a.warm)
    t0 = time.perf_counter()
    comp, wall = t.run(a.steps)
    if a.fp32:
        desc = desc.replace("fp64", "fp32")
    print(f"{desc}: {a.steps} steps compute {comp*1e3:.3f} ms wall {wall*1e3:.3f} ms "
          f"-> {n*m*l*a.steps/wall/1e9:.2f} Gcell/s, launches {t.launches}")
