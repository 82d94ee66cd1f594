#!/bin/bash
# fp32 two-rows-per-warp variants at l = 128: bit-identity check, then A/B timing.
mkdir -p gpurun_out
for v in f32rw2 f32rw2b; do
  echo "== $v" ; IMB_LIB=$PWD/experiments/libimb_$v.so timeout 300 python tools/fp32_check.py 2>&1 | tail -8
done > gpurun_out/rw2_check.txt 2>&1
timeout 900 python tools/ab.py --fp32 --configs c4,c5s --reps 3 --steps 10 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,rw2=experiments/libimb_f32rw2.so,rw2b=experiments/libimb_f32rw2b.so \
  > gpurun_out/rw2_ab.txt 2>&1
cat gpurun_out/rw2_check.txt gpurun_out/rw2_ab.txt
