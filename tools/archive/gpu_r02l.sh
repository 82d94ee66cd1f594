#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_m.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_m.log
IMB_LIB=$PWD/experiments/libimb_k4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "config2 or matrix" > gpurun_out/pytest_m_k4.log 2>&1; echo pytest_k4=$?; tail -2 gpurun_out/pytest_m_k4.log
python tools/ab.py --configs c4,c5d --reps 3 --libs prev=experiments/libimb_prev.so,cur=paper_1507_01265_b200/libimb_b200.so,k4=experiments/libimb_k4.so > gpurun_out/ab_m.txt 2>&1
cat gpurun_out/ab_m.txt
