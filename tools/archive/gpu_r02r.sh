#!/bin/bash
# Parity margins at every BASELINE config's full grid and step count (the
# product), then the same for a fp32 build with FMA contraction (experiment).
mkdir -p gpurun_out
python tools/parity_margin.py --configs c1,c2,c4,c4s,c5d,c5s --out gpurun_out/r02_parity_margins.jsonl > gpurun_out/margins_r.log 2>&1; echo margins=$?
cat gpurun_out/margins_r.log
IMB_LIB=$PWD/experiments/libimb_fma32.so python tools/parity_margin.py --configs c4s,c5s --out gpurun_out/r02_parity_margins_fma32.jsonl > gpurun_out/margins_fma.log 2>&1; echo margins_fma=$?
cat gpurun_out/margins_fma.log
python tools/ab.py --fp32 --configs c4,c5s --reps 3 --libs exact=paper_1507_01265_b200/libimb_b200.so,fma=experiments/libimb_fma32.so > gpurun_out/ab_r.txt 2>&1
cat gpurun_out/ab_r.txt
