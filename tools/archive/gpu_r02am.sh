#!/bin/bash
# fp32 XR: both outermost rows' donors on warp 0 (phase B balance); parity + A/B
mkdir -p gpurun_out
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_am.log 2>&1; echo fp32_check=$?; cat gpurun_out/fp32_check_am.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_am.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_am.log
python tools/ab.py --fp32 --configs c4,c5s --reps 3 --libs xr2=experiments/libimb_xr2.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_am.txt 2>&1
cat gpurun_out/ab_am.txt
