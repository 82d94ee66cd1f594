#!/usr/bin/env python3
"""Small MPDATA runs for compute-sanitizer.

Each case drives one kernel family through the C-ABI on a grid small enough
for racecheck/synccheck: the fused step (fp64 two-segment rows, fp32, plain
IORD=2, the IORD=3 pair of launches, l = 32/64 tiles), the staged kernels,
the self-pushing periodic slab and an in-process group whose fused steps push
edge planes into each other's halos. Run as

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py CASE
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1507_01265_b200 import mpdata  # noqa: E402

O = mpdata.Options
CASES = {
    # name: (n, m, l, options, steps, group shares or None)
    "fused_f64": (8, 20, 128, O(2, True, True), 2, None),
    "fused_f32": (8, 20, 128, O(2, True, False), 2, None),
    "fused_plain": (6, 20, 128, O(2, False, True), 2, None),
    "fused_iord3": (12, 20, 128, O(3, True, True), 1, None),
    "fused_l64": (8, 36, 64, O(2, True, True), 2, None),
    "fused_l32": (8, 70, 32, O(2, False, True), 2, None),
    "staged": (8, 12, 24, O(2, True, True), 2, None),
    "group": (12, 20, 128, O(2, True, True), 2, [4, 3, 5]),
    "group_flags": (12, 20, 128, O(2, True, False), 2, [5, 3, 4]),
}


def run(name: str) -> None:
    n, m, l, opts, steps, shares = CASES[name]
    if shares is None:
        with mpdata.Team(n, m, l, opts) as t:
            t.init_recipe(mpdata.RECIPE_ROTCUBE, 42)
            t.run(steps)
            t.download("x")
    else:
        g = mpdata.Group(n, m, l, shares, opts=opts)
        try:
            g.init_recipe(mpdata.RECIPE_ROTCUBE, 42)
            if name.endswith("_flags"):
                g.set_sync("flags")
            g.run(steps)
            g.download("x")
        finally:
            g.close()
    print(f"{name} ok")


if __name__ == "__main__":
    for arg in sys.argv[1:] or sorted(CASES):
        run(arg)
