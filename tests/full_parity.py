"""Full-size oracle parity of the BASELINE configs (shared by
tests/test_full_size_parity.py and tools/parity_margin.py).

The GPU team generates the seeded recipe on the device (bit-identical to the
host recipe, tests/test_gpu_parity.py::test_device_init_is_bit_identical_to_host);
the five fields are downloaded and handed to the CPU oracle, so both sides
step exactly the same bytes. Errors are measured plane-chunked (no multi-GB
temporaries): the per-cell relative error |gpu - ref| / max(|ref|, 1)
(the north_star tolerance), the normwise
max|gpu - ref| / max|ref|, and the count of bit-identical cells.
"""
from __future__ import annotations

import os
import time

import numpy as np

# name -> (n, m, l, iord, nonos, fp64, recipe, steps)
CONFIGS = {
    "c1": (64, 64, 32, 2, False, True, 1, 10),
    "c2": (256, 256, 64, 2, True, True, 2, 50),
    "c4": (1024, 512, 128, 2, True, True, 2, 100),
    "c4s": (1024, 512, 128, 2, True, False, 2, 100),
    "c5d": (2048, 1024, 128, 3, True, True, 2, 100),
    "c5s": (2048, 1024, 128, 3, True, False, 2, 100),
}
TOL = {True: 1e-12, False: 1e-5}


def errors(got: np.ndarray, want: np.ndarray, chunk: int = 32) -> dict:
    worst, num, den, same = 0.0, 0.0, 0.0, 0
    for i in range(0, want.shape[0], chunk):
        a = got[i:i + chunk].astype(np.float64)
        b = want[i:i + chunk].astype(np.float64)
        d = np.abs(a - b)
        worst = max(worst, float(np.max(d / np.maximum(np.abs(b), 1.0))))
        num = max(num, float(np.max(d)))
        den = max(den, float(np.max(np.abs(b))))
        same += int(np.count_nonzero(got[i:i + chunk] == want[i:i + chunk]))
    return {"max_rel_err": worst, "normwise_rel_err": num / den if den else num,
            "bit_identical_frac": same / want.size}


def run_config(name: str, steps: int | None = None, threads: int | None = None,
               seed: int = 42) -> dict:
    from oracle import oracle as O
    from paper_1507_01265_b200.mpdata import Options, Team

    n, m, l, iord, nonos, fp64, recipe, full = CONFIGS[name]
    steps = full if steps is None else steps
    threads = threads or os.cpu_count() or 1
    opts = Options(iord, nonos, fp64)
    with Team(n, m, l, opts) as t:
        t.init_recipe(recipe, seed)
        fields = [t.download(f) for f in "xuvwh"]
        t0 = time.perf_counter()
        t.run(steps)
        gpu_s = time.perf_counter() - t0
        got = t.download("x")
        launches = t.launches
    t0 = time.perf_counter()
    want = O.run(*fields, iord=iord, nonos=nonos, steps=steps, threads=threads)
    cpu_s = time.perf_counter() - t0
    del fields
    rec = {"config": name, "grid": [n, m, l], "iord": iord, "nonos": nonos,
           "dtype": "f64" if fp64 else "f32", "steps": steps, "seed": seed, "tolerance": TOL[fp64],
           "oracle_threads": threads, "oracle_s": round(cpu_s, 2), "gpu_s": round(gpu_s, 3),
           "gpu_launches": launches, "min_ref": float(want.min()), "max_ref": float(want.max())}
    rec.update(errors(got, want))
    rec["pass"] = rec["max_rel_err"] <= TOL[fp64]
    return rec
