#!/bin/bash
mkdir -p gpurun_out/cs
timeout 1500 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 --libs base=paper_1507_01265_b200/libimb_b200.so,outcs=experiments/libimb_outcs.so,m2na=experiments/libimb_m2na.so,both=experiments/libimb_both.so > gpurun_out/cs/ab2.txt 2>&1
timeout 1500 python tools/ab.py --fp32 --configs c4,c5s --reps 3 --steps 20 --libs base=paper_1507_01265_b200/libimb_b200.so,outcs=experiments/libimb_outcs.so,m2na=experiments/libimb_m2na.so >> gpurun_out/cs/ab2.txt 2>&1
cat gpurun_out/cs/ab2.txt
