"""Generates the committed golden fixtures (run here, where /root/reference exists).

* mpdata_checksums.json — FNV-1a checksums of the MPDATA oracle on small
  seeded cases (the golden-checksum file SPEC.md:274/:311 asks for; the
  reference never produced one).
* partition_ref.json — outputs of the UNMODIFIED reference partitioner
  (oracle/_ref/libimb_ref.so built from /root/reference/proj/src) on the
  paper's worked example, the SURVEY Appendix B cases and seeded random
  tables, so parity can be checked even where the reference is absent.

    python tests/golden/make_golden.py
"""
import json
import random
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

HERE = Path(__file__).resolve().parent


def mpdata_rows():
    cases = [
        (1, (64, 64, 32), 2, False, 10, "fp64"),   # config 1
        (2, (32, 32, 16), 2, True, 5, "fp64"),     # config-2 recipe, small
        (2, (24, 16, 16), 3, True, 4, "fp64"),     # config-5 scheme, small
        (2, (24, 16, 16), 3, True, 4, "fp32"),
        (0, (16, 12, 10), 1, False, 3, "fp64"),
        (0, (8, 8, 8), 2, True, 3, "fp64"),        # SPEC.md:274 8x8x8 seed 42
    ]
    rows = []
    for recipe, grid, iord, nonos, steps, prec in cases:
        dt = np.float64 if prec == "fp64" else np.float32
        f = O.init_fields(recipe, *grid, seed=42, dtype=dt)
        y = O.run(*f, iord=iord, nonos=nonos, steps=steps, threads=4)
        rows.append(dict(recipe=recipe, grid=list(grid), iord=iord, nonos=nonos, steps=steps,
                         precision=prec, seed=42, checksum=f"{O.checksum(y):016x}"))
    return rows


PAPER = dict(unit=15360, g=8, samples=[(112, 1436742.0), (120, 1240377.0), (128, 1418579.0)])


def random_table(rng, n_max=40):
    g = rng.choice([1, 1, 2, 4])
    unit = rng.choice([1, 7, 15360, 65536])
    x = rng.randint(1, 4) * g
    samples = []
    for _ in range(rng.randint(1, 9)):
        samples.append((x, rng.uniform(0.5, 100.0) * (1e6 if unit > 1000 else 1.0)))
        x += rng.randint(1, 3) * g
    total = rng.randint(1, n_max // g) * g
    p = rng.randint(1, 5)
    return dict(unit=unit, g=g, samples=samples, total=total, p=p,
                allow_idle=rng.random() < 0.25)


def gpu_like_table():
    xs = [8, 16, 32, 64, 128, 256, 512, 1024, 2048]
    sp = [20e9, 31e9, 44e9, 53e9, 60e9, 64e9, 67e9, 69e9, 70.5e9]
    return dict(unit=512 * 128, g=8, samples=list(zip(xs, sp)))


def partition_rows():
    rows = []

    def add(kind, t, total, p, allow_idle=False):
        st, sh, pt, ms, off = O.ref_partition(kind, t["unit"], t["g"], t["samples"], total, p,
                                              allow_idle)
        rows.append(dict(kind=kind, unit=t["unit"], g=t["g"], samples=t["samples"], total=total,
                         p=p, allow_idle=allow_idle, status=st, shares=sh, per_time=pt,
                         makespan=ms, offset=off))

    for kind in ("paired", "general", "brute"):
        add(kind, PAPER, 480, 4)
    add("paired", PAPER, 480, 3)  # ContractError
    add("paired", PAPER, 484, 4)  # AlignmentError
    t1 = dict(unit=1, g=1, samples=[(1, 1), (2, 4), (3, 3), (4, 4), (5, 5), (6, 6)])
    add("general", t1, 6, 3)
    add("brute", t1, 6, 3)
    t2 = dict(unit=1, g=1, samples=[(1, 1), (2, 8), (3, 3), (4, 4)])
    add("general", t2, 4, 4, True)
    add("brute", t2, 4, 4, True)
    t3 = dict(unit=1, g=1, samples=[(x, 5.0) for x in range(1, 11)])
    add("general", t3, 10, 4)
    add("brute", t3, 10, 4)
    gt = gpu_like_table()
    for p in (1, 2, 4, 8):
        add("general", gt, 2048, p)
        if p % 2 == 0:
            add("paired", gt, 2048, p)
    rng = random.Random(20251020)
    for _ in range(300):
        t = random_table(rng)
        for kind in ("paired", "general", "brute"):
            add(kind, t, t["total"], t["p"], t["allow_idle"])
    return rows


if __name__ == "__main__":
    (HERE / "mpdata_checksums.json").write_text(json.dumps(mpdata_rows(), indent=1) + "\n")
    (HERE / "partition_ref.json").write_text(json.dumps(partition_rows()) + "\n")
    print("wrote", HERE / "mpdata_checksums.json", HERE / "partition_ref.json")
