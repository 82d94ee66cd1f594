#!/usr/bin/env python3
"""Per-chunk timeline of the host-buffer step (IMB_PIPE_TRACE=1): C4 fp64, pinned buffers.

    IMB_PIPE_TRACE=1 python tools/pipe_trace.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402  (pinned host buffers)

from bench import CONFIGS  # noqa: E402
from paper_1507_01265_b200 import mpdata  # noqa: E402

n, m, l, iord, nonos, fp64, recipe, _ = CONFIGS["c4"]
with mpdata.Team(n, m, l, mpdata.Options(iord, nonos, fp64)) as t:
    t.init_recipe(recipe, 42)
    xin = torch.empty(t.shape, dtype=torch.float64, pin_memory=True).numpy()
    xout = torch.empty(t.shape, dtype=torch.float64, pin_memory=True).numpy()
    xin[...] = t.download("x")
    for i in range(4):
        a = time.perf_counter()
        t.step_host(xin, xout)
        print(f"step {i}: {(time.perf_counter() - a) * 1e3:.2f} ms wall", file=sys.stderr, flush=True)
        xin, xout = xout, xin
