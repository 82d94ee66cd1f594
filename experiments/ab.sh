#!/bin/bash
# A/B: product library vs experiments/libimb_variants.so on c4/c2/c5d, fp64 and fp32.
for rep in 1 2; do
for cfg in ${CFGS:-c4 c2 c5d}; do
  for fp in "" "--fp32"; do
    echo -n "A $cfg $fp: "; python tools/profile_step.py --config $cfg $fp --warm 3 --steps 20 2>&1 | tail -1 | sed 's/.*-> //'
    echo -n "B $cfg $fp: "; IMB_LIB=$PWD/experiments/libimb_variants.so python tools/profile_step.py --config $cfg $fp --warm 3 --steps 20 2>&1 | tail -1 | sed 's/.*-> //'
  done
done
done
