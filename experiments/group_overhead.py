"""Decomposition overhead on one GPU: a periodic single slab vs the same grid
as P slabs in one process (in-process ring, halos pushed by the step kernel,
event or flag synchronisation). All slabs share the GPU, so equal totals mean
the ring protocol costs nothing measurable."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1507_01265_b200 import mpdata  # noqa: E402

n, m, l, steps = 1024, 512, 128, 20
opts = mpdata.Options(2, True, True)
with mpdata.Team(n, m, l, opts) as t:
    t.init_recipe(2, 42)
    t.run(3)
    _, wall = t.run(steps)
print(f"single slab: {n*m*l*steps/wall/1e9:.2f} Gcell/s")
for shares in ([512, 512], [256] * 4, [128] * 8):
    for sync in ("events", "flags"):
        g = mpdata.Group(n, m, l, shares, opts=opts)
        g.set_sync(sync)
        g.init_recipe(2, 42)
        g.run(3)
        _, wall = g.run(steps)
        g.close()
        print(f"{len(shares)} slabs, {sync}: {n*m*l*steps/wall/1e9:.2f} Gcell/s")
