#!/bin/bash
# fp64 limiter in/out sums as sum|f| +- (left - right): speed A/B and 100-step parity margins
mkdir -p gpurun_out
python tools/ab.py --configs c4,c5d --reps 3 --libs head=experiments/libimb_head.so,sd=experiments/libimb_sd.so > gpurun_out/ab_ae.txt 2>&1
cat gpurun_out/ab_ae.txt
IMB_LIB=$PWD/experiments/libimb_sd.so timeout 900 python tools/parity_margin.py --configs c4,c5d > gpurun_out/margin_sd.txt 2>&1; cat gpurun_out/margin_sd.txt
