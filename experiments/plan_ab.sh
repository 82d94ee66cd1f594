#!/bin/bash
echo "== new plan"; python experiments/slabs.py
echo "== old plan"; IMB_LIB=$PWD/experiments/libimb_variants.so python experiments/slabs.py
for cfg in c5d c2; do for fp in "" "--fp32"; do
  echo -n "$cfg$fp new: "; python tools/profile_step.py --config $cfg $fp --warm 3 --steps 10 | sed 's/.*-> //'
  echo -n "$cfg$fp old: "; IMB_LIB=$PWD/experiments/libimb_variants.so python tools/profile_step.py --config $cfg $fp --warm 3 --steps 10 | sed 's/.*-> //'
done; done
