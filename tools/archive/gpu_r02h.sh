#!/bin/bash
mkdir -p gpurun_out
IMB_LIB=$PWD/experiments/libimb_two.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo pytest_two=$?; tail -2 gpurun_out/pytest_h.log
python tools/ab.py --configs c4,c5d --reps 3 --libs cur=paper_1507_01265_b200/libimb_b200.so,two=experiments/libimb_two.so > gpurun_out/ab_h.txt 2>&1
cat gpurun_out/ab_h.txt
