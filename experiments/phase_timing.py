"""Run C4 steps with the timing build and print per-phase cycle shares."""
import ctypes as C
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
os.environ["IMB_LIB"] = str(ROOT / "experiments" / "libimb_timing.so")
sys.path.insert(0, str(ROOT))
from paper_1507_01265_b200 import _lib, mpdata  # noqa: E402
lib = _lib.load()
f = lib.imb_debug_phase_cycles
buf = (C.c_ulonglong * 10)()
for cfg in [(1024, 512, 128, True), (1024, 512, 128, False)]:
    n, m, l, fp64 = cfg
    with mpdata.Team(n, m, l, mpdata.Options(2, True, fp64)) as t:
        t.init_recipe(2, 42)
        t.run(2)
        f(buf, 1)
        comp, wall = t.run(5)
        f(buf, 1)
    names = ["donor", "sync1", "pseudo", "sync2", "beta", "sync3", "limit+final", "sync4"]
    tot = sum(buf[i] for i in range(8))
    print(f"fp64={fp64}: {n*m*l*5/wall/1e9:.2f} Gcell/s;",
          ", ".join(f"{nm} {100*buf[i]/tot:.1f}%" for i, nm in enumerate(names)))
