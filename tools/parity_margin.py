"""Parity margins of the GPU path against the CPU oracle at the BASELINE
configs' full grids and step counts (fp64 and fp32).

    python tools/parity_margin.py [--configs c1,c2,c4,c4s,c5d,c5s] [--steps N] [--seeds 42,7]
                                  [--out profiles/r02_parity_margins.jsonl]

One JSON line per config: max per-cell relative error (|ref| floored at 1),
normwise error, the fraction of bit-identical cells, the north_star
tolerance and the oracle/GPU wall times.
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from tests.full_parity import CONFIGS, run_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c4,c4s,c5d,c5s")
    ap.add_argument("--steps", type=int, default=None, help="override every config's step count")
    ap.add_argument("--seeds", default="42", help="comma-separated recipe seeds")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    out = open(a.out, "a") if a.out else None
    ok = True
    for name in a.configs.split(","):
        if name not in CONFIGS:
            raise SystemExit(f"unknown config {name}")
        for seed in (int(v) for v in a.seeds.split(",")):
            rec = run_config(name, a.steps, seed=seed)
            ok = ok and rec["pass"]
            line = json.dumps(rec)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
