import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle as O
from paper_1507_01265_b200.mpdata import Team, Options
for cfg, steps, nonos in (((256, 256, 64), 50, True), ((64, 64, 32), 10, False)):
    f = O.init_fields(2 if nonos else 1, *cfg, seed=42)
    with Team(*cfg, Options(2, nonos, True)) as t:
        t.upload_all(*f); t.run(steps); got = t.download("x")
    want = O.run(*f, iord=2, nonos=nonos, steps=steps, threads=8)
    err = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0)))
    print(cfg, steps, "max rel err", err)
