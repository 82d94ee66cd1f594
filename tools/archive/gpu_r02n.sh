#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_n.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_n.log
python tools/ab.py --configs c5d --reps 3 --libs prev=experiments/libimb_prev.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_n.txt 2>&1
cat gpurun_out/ab_n.txt
