#!/bin/bash
export IMB_LIB=$PWD/experiments/libimb_variants.so
for v in 12 14 20; do
  echo "IMB_NW=$v"; export IMB_NW=$v
  python tools/profile_step.py --config c4 --warm 2 --steps 10
  python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10
done
