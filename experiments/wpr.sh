#!/bin/bash
export IMB_LIB=$PWD/experiments/libimb_variants.so
for v in "" 1; do
  echo "IMB_WPR2=$v"
  if [ -n "$v" ]; then export IMB_WPR2=1; else unset IMB_WPR2; fi
  python tools/profile_step.py --config c4 --warm 2 --steps 10
  python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10
done
