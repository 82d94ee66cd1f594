#!/bin/bash
# XR: two extra halo rows per tile handled by warps 0 and 15 (14-row tiles): parity + A/B
mkdir -p gpurun_out
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_af.log 2>&1; echo fp32_check=$?; cat gpurun_out/fp32_check_af.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_af.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_af.log
python tools/ab.py --configs c4,c5d,c2 --reps 3 --libs head=experiments/libimb_head.so,xr=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_af.txt 2>&1
python tools/ab.py --fp32 --configs c4,c5s --reps 2 --libs head=experiments/libimb_head.so,xr=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/ab_af.txt 2>&1
cat gpurun_out/ab_af.txt
