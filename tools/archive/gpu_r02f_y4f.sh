#!/bin/bash
# fp32: extra y-face one element each on four warps (IMB_XR_Y4_F32): bit identity, A/B
mkdir -p gpurun_out/y4f
for v in y4f y4f2 y4f3; do echo "== $v"; IMB_LIB=$PWD/experiments/libimb_$v.so timeout 300 python tools/fp32_check.py 2>&1 | tail -6; done > gpurun_out/y4f/check.txt 2>&1
cat gpurun_out/y4f/check.txt
timeout 1500 python tools/ab.py --fp32 --configs c4,c5s --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,y4f=experiments/libimb_y4f.so,y4f2=experiments/libimb_y4f2.so,y4f3=experiments/libimb_y4f3.so > gpurun_out/y4f/ab.txt 2>&1
cat gpurun_out/y4f/ab.txt
