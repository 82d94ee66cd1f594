#!/bin/bash
# placement / saving knobs re-measured on the three-slot kernel
mkdir -p gpurun_out/retune
timeout 1500 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,yw1=experiments/libimb_yw1.so,nobc=experiments/libimb_nobc.so,nolf=experiments/libimb_nolf.so,k3=experiments/libimb_k3.so,xm7=experiments/libimb_xm7.so,sp5=experiments/libimb_sp5.so > gpurun_out/retune/ab.txt 2>&1
cat gpurun_out/retune/ab.txt
