#!/bin/bash
# Device-resident step throughput of every BASELINE config (fp64, and fp32 where the
# config allows), one B200, product build. Output: profiles/r01_configs.txt format.
for cfg in c1 c2 c4 c5d c5s; do
  python tools/profile_step.py --config $cfg --warm 5 --steps 30 | sed "s/^/$cfg fp64-or-native: /"
done
for cfg in c2 c4; do
  python tools/profile_step.py --config $cfg --fp32 --warm 5 --steps 30 | sed "s/^/$cfg fp32: /"
done
