#!/bin/bash
mkdir -p gpurun_out/k3
timeout 1200 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,k3=experiments/libimb_k3.so,mm2=experiments/libimb_mm2.so \
  > gpurun_out/k3/ab.txt 2>&1
cat gpurun_out/k3/ab.txt
