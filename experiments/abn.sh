#!/bin/bash
# Interleaved A/B/n: the working-tree library vs experiments/libimb_<name>.so for each
# name in $LIBS, on $CFGS (default c4) and $FPS (fp64 and/or fp32), $REPS rounds.
for rep in $(seq ${REPS:-2}); do
  for cfg in ${CFGS:-c4}; do
    for fp in ${FPS:-fp64}; do
      flag=""; [ "$fp" = fp32 ] && flag="--fp32"
      echo -n "cur $cfg $fp: "; python tools/profile_step.py --config $cfg $flag --warm 3 --steps ${STEPS:-20} 2>&1 | tail -1 | sed 's/.*-> //'
      for n in $LIBS; do
        echo -n "$n $cfg $fp: "; IMB_LIB=$PWD/experiments/libimb_$n.so python tools/profile_step.py --config $cfg $flag --warm 3 --steps ${STEPS:-20} 2>&1 | tail -1 | sed 's/.*-> //'
      done
    done
  done
done
