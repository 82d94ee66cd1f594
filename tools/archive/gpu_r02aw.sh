#!/bin/bash
# re-test instruction-count options on the extra-rows layout: shared-compare extrema (fp64), packed fp32
mkdir -p gpurun_out
python tools/ab.py --configs c4,c5d --reps 3 --libs cur=paper_1507_01265_b200/libimb_b200.so,mm2=experiments/libimb_mm2.so > gpurun_out/ab_aw.txt 2>&1
python tools/ab.py --fp32 --configs c4,c5s --reps 3 --libs cur=paper_1507_01265_b200/libimb_b200.so,pk=experiments/libimb_pk.so >> gpurun_out/ab_aw.txt 2>&1
cat gpurun_out/ab_aw.txt
