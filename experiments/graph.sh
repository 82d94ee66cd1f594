#!/bin/bash
# CUDA-graph step pairs on vs off (IMB_GRAPH=0), all configs.
for cfg in c1 c2 c4; do
  for g in 1 0; do echo -n "graph=$g $cfg: "; IMB_GRAPH=$g python tools/profile_step.py --config $cfg --warm 4 --steps 40 | sed 's/.*-> //'; done
done
