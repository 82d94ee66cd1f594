#!/bin/bash
# Split (two-kernel) IORD=2 step vs the fused kernel.
for cfg in c4 c2; do for fp in "" "--fp32"; do
  for sp in 0 1; do echo -n "$cfg$fp split=$sp: "; IMB_SPLIT=$sp python tools/profile_step.py --config $cfg $fp --warm 3 --steps 20 | sed 's/.*-> //'; done
done; done
