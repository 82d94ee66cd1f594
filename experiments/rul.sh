#!/bin/bash
# ptxas --register-usage-level sweep (default 5 = product build).
for lvl in 5 0 2 8 10; do
  L=$PWD/experiments/libimb_rul$lvl.so; [ $lvl = 5 ] && L=$PWD/paper_1507_01265_b200/libimb_b200.so
  for fp in "" "--fp32"; do echo -n "rul$lvl c4$fp: "; IMB_LIB=$L python tools/profile_step.py --config c4 $fp --warm 3 --steps 20 | sed 's/.*-> //'; done
done
