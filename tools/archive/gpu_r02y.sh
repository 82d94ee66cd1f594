#!/bin/bash
# MODE 2 (IORD=3 pass 3) L2 prefetch of the bounds planes: A/B on C5 fp64
mkdir -p gpurun_out
python tools/ab.py --configs c5d --reps 4 --libs head=experiments/libimb_head.so,cur=paper_1507_01265_b200/libimb_b200.so,m2pf0=experiments/libimb_m2pf0.so > gpurun_out/ab_y.txt 2>&1
cat gpurun_out/ab_y.txt
