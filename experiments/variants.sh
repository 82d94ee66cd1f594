#!/bin/bash
export IMB_LIB=$PWD/experiments/libimb_variants.so
for v in ${VARS:-10 11 20 21 40 41}; do
  echo "variant $v"
  for fp in "" "--fp32"; do IMB_FUSED_VARIANT=$v python tools/profile_step.py --config c4 $fp --warm 2 --steps 10; done
done
