#!/bin/bash
# L2 bulk-prefetch distance sweep (IMB_PF planes ahead; 0 = off).
for pf in ${PFS:-0 1 2 3 4 6 8}; do
  for cfg in c4 c5d; do
    for fp in "" "--fp32"; do echo -n "pf=$pf $cfg $fp: "; IMB_PF=$pf python tools/profile_step.py --config $cfg $fp --warm 2 --steps 10; done
  done
done
