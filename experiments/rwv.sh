#!/bin/bash
# Two-rows-per-warp tile variants (IMB_RWV, experiments/libimb_variants.so).
export IMB_LIB=$PWD/experiments/libimb_variants.so
for v in 0 1 2 3 4 7 5 6; do
  for fp in "" "--fp32"; do echo -n "rwv=$v $fp: "; IMB_RWV=$v python tools/profile_step.py --config c4 $fp --warm 2 --steps 20 2>&1 | tail -1; done
done
