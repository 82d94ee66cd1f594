#!/bin/bash
# C5 fp64 re-tests on the streaming-store build: XR in pass 2 (xm7), three psi^(1) slots in pass 2 (x13m3) / pass 3 (x13m5)
mkdir -p gpurun_out/c5re
timeout 1500 python tools/ab.py --configs c5d --reps 3 --steps 10 --libs base=paper_1507_01265_b200/libimb_b200.so,xm7=experiments/libimb_xm7.so,x13m3=experiments/libimb_x13m3.so,x13m5=experiments/libimb_x13m5.so > gpurun_out/c5re/ab.txt 2>&1
cat gpurun_out/c5re/ab.txt
