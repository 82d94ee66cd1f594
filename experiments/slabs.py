"""Per-slab throughput for the slab thicknesses an N-GPU C4 run gives each GPU."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1507_01265_b200 import mpdata  # noqa: E402
for fp64 in (True, False):
    for n in (128, 256, 512, 1024):
        with mpdata.Team(n, 512, 128, mpdata.Options(2, True, fp64)) as t:
            t.init_recipe(2, 42)
            t.run(3)
            _, wall = t.run(20)
        print(f"fp64={fp64} n={n}: {n*512*128*20/wall/1e9:.2f} Gcell/s", flush=True)
