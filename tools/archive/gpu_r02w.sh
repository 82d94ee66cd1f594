#!/bin/bash
# compiler-flag variants of the whole library, interleaved A/B on C4 fp64 / C5 fp64 / C4 fp32
mkdir -p gpurun_out
L=head=experiments/libimb_head.so,xo=experiments/libimb_xo.so,dv=experiments/libimb_dv.so,o2=experiments/libimb_o2.so
python tools/ab.py --configs c4,c5d --reps 3 --libs $L > gpurun_out/ab_w.txt 2>&1
python tools/ab.py --fp32 --configs c4 --reps 2 --libs $L >> gpurun_out/ab_w.txt 2>&1
cat gpurun_out/ab_w.txt
