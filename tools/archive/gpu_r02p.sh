#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "iord3 or matrix or IORD or scheme" > gpurun_out/pytest_p.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_p.log
python tools/ab.py --configs c5d --reps 3 --libs prev=experiments/libimb_prev.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_p.txt 2>&1
python tools/ab.py --fp32 --configs c5s --reps 3 --libs prev=experiments/libimb_prev.so,cur=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/ab_p.txt 2>&1
cat gpurun_out/ab_p.txt
