#!/bin/bash
# XR_DEFER: the extra row's y-face computed one plane ahead in the donor phase; parity + A/B
mkdir -p gpurun_out
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_ai.log 2>&1; echo fp32_check=$?; tail -3 gpurun_out/fp32_check_ai.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_ai.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ai.log
python tools/ab.py --configs c4,c5d --reps 3 --libs xr=experiments/libimb_xr.so,defer=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_ai.txt 2>&1
python tools/ab.py --fp32 --configs c4,c5s --reps 2 --libs xr=experiments/libimb_xr.so,defer=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/ab_ai.txt 2>&1
cat gpurun_out/ab_ai.txt
