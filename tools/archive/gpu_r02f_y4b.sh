#!/bin/bash
mkdir -p gpurun_out/y4
python experiments/phase_timing.py > gpurun_out/y4/phase_timing.txt 2>&1; cat gpurun_out/y4/phase_timing.txt
timeout 1500 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,m5=experiments/libimb_y4m5.so > gpurun_out/y4/ab_m5.txt 2>&1
cat gpurun_out/y4/ab_m5.txt
