#!/bin/bash
mkdir -p gpurun_out/seam
timeout 1500 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 --libs base=paper_1507_01265_b200/libimb_b200.so,seam=experiments/libimb_seam.so > gpurun_out/seam/ab.txt 2>&1
cat gpurun_out/seam/ab.txt
