#!/bin/bash
# XR for l = 64 (two rows per warp, 34 region rows): parity + A/B on C2
mkdir -p gpurun_out
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_aj.log 2>&1; echo fp32_check=$?; tail -4 gpurun_out/fp32_check_aj.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_aj.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_aj.log
python tools/ab.py --configs c2 --reps 3 --steps 50 --libs xr=experiments/libimb_xr.so,xr64=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_aj.txt 2>&1
python tools/ab.py --fp32 --configs c2 --reps 3 --steps 50 --libs xr=experiments/libimb_xr.so,xr64=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/ab_aj.txt 2>&1
cat gpurun_out/ab_aj.txt
