"""Run C4 steps with the timing build and print per-phase cycle shares per warp
(warp w owns region row w+1 with the extra halo rows (Cfg::XR): rows 0,1 and 16,17 are the recomputed j-halo)."""
import ctypes as C
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
os.environ["IMB_LIB"] = str(ROOT / "experiments" / "libimb_timing.so")
sys.path.insert(0, str(ROOT))
from paper_1507_01265_b200 import _lib, mpdata  # noqa: E402
lib = _lib.load()
buf = (C.c_ulonglong * 320)()
slots = [(2, "pseudo"), (3, "bar1"), (4, "beta"), (5, "bar2"), (6, "lim+fin"), (8, "donor"),
         (7, "bar3")]
for n, m, l, fp64 in [(1024, 512, 128, True), (1024, 512, 128, False)]:
    f = lib.imb_debug_phase_cycles if fp64 else lib.imb_debug_phase_cycles_f32
    with mpdata.Team(n, m, l, mpdata.Options(2, True, fp64)) as t:
        t.init_recipe(2, 42)
        t.run(2)
        f(buf, 1)
        comp, wall = t.run(5)
        f(buf, 1)
    print(f"fp64={fp64}: {n*m*l*5/wall/1e9:.2f} Gcell/s (timing build)")
    print("warp " + " ".join(f"{nm:>8}" for _, nm in slots))
    tot = sum(buf[s * 32 + w] for s, _ in slots for w in range(16)) / 16
    for w in range(16):
        print(f"{w:4d} " + " ".join(f"{100 * buf[s * 32 + w] / tot:8.1f}" for s, _ in slots))
    print("all  " + " ".join(f"{100 * sum(buf[s * 32 + w] for w in range(16)) / 16 / tot:8.1f}"
                             for s, _ in slots))
