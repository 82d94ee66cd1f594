#!/bin/bash
V=$PWD/experiments/libimb_variants.so
for rep in 1 2; do
  for pf in 0 1 2; do echo -n "pf=$pf c4: "; IMB_PF=$pf python tools/profile_step.py --config c4 --warm 3 --steps 20 | sed 's/.*-> //'; done
  for pf in 0 1; do echo -n "pf=$pf c5d: "; IMB_PF=$pf python tools/profile_step.py --config c5d --warm 3 --steps 10 | sed 's/.*-> //'; done
  for v in 8 9; do echo -n "fp32 v$v c4: "; IMB_LIB=$V IMB_RWV=$v python tools/profile_step.py --config c4 --fp32 --warm 3 --steps 20 | sed 's/.*-> //'; done
done
