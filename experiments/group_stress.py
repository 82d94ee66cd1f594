"""300-step in-process rings (event and flag sync) against one slab: bit-identical."""
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1507_01265_b200 import mpdata
for shares, opts in (([9, 7, 16], mpdata.Options(2, True, True)), ([8] * 4, mpdata.Options(3, True, False))):
    n = sum(shares)
    with mpdata.Team(n, 20, 64, opts) as t:
        t.init_recipe(2, 5); t.run(300); want = t.download("x")
    for sync in ("events", "flags"):
        g = mpdata.Group(n, 20, 64, shares, opts=opts); g.set_sync(sync); g.init_recipe(2, 5)
        g.run(100); g.run(200)
        print(shares, sync, np.array_equal(g.download("x"), want)); g.close()
