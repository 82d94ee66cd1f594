#!/bin/bash
# three psi^(1) slots (IMB_X1_3 mask over MODE): x4 = none, m1 = MODE 0 (default build), m3 = MODE 0+1, m7 = all
mkdir -p gpurun_out/x13
timeout 1200 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs x4=experiments/libimb_x4.so,m1=paper_1507_01265_b200/libimb_b200.so,m3=experiments/libimb_x13m3.so,m7=experiments/libimb_x13m7.so > gpurun_out/x13/ab_c.txt 2>&1
cat gpurun_out/x13/ab_c.txt
