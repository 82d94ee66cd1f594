#!/bin/bash
# fp32: row 17's donor on a scheduler-0 warp other than warp 0 (4, 8, 12)
mkdir -p gpurun_out
IMB_LIB=$PWD/experiments/libimb_d17w12.so timeout 600 python tools/fp32_check.py 2>&1 | tail -4
python tools/ab.py --fp32 --configs c4 --reps 3 --libs cur=paper_1507_01265_b200/libimb_b200.so,w12=experiments/libimb_d17w12.so,w8=experiments/libimb_d17w8.so,w4=experiments/libimb_d17w4.so > gpurun_out/ab_as.txt 2>&1
cat gpurun_out/ab_as.txt
