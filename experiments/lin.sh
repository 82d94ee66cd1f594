#!/bin/bash
# Linear (tile, plane) split vs grid split; B = previous build (experiments/libimb_variants.so).
V=$PWD/experiments/libimb_variants.so
for cfg in c4 c5d; do for fp in "" "--fp32"; do
  echo -n "$cfg$fp old: "; IMB_LIB=$V python tools/profile_step.py --config $cfg $fp --warm 3 --steps 20 | sed 's/.*-> //'
  for l in 0 1; do echo -n "$cfg$fp lin=$l: "; IMB_LINSPLIT=$l python tools/profile_step.py --config $cfg $fp --warm 3 --steps 20 | sed 's/.*-> //'; done
done; done
for n in 128 256 512; do
  python - <<PY
import sys, os
sys.path.insert(0, ".")
from paper_1507_01265_b200 import mpdata
for lin in ("0", "1"):
    pass
PY
done
