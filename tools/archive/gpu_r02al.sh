#!/bin/bash
# final XR layout (fp64 MODE 0 splits the extra y-face over warps 0/15): parity + A/B vs the first XR build
mkdir -p gpurun_out
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_al.log 2>&1; echo fp32_check=$?; tail -2 gpurun_out/fp32_check_al.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_checked.py tests/test_full_size_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_al.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_al.log
python tools/ab.py --configs c4,c5d --reps 3 --libs xr=experiments/libimb_xr.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_al.txt 2>&1
python tools/ab.py --fp32 --configs c4,c5s --reps 2 --libs xr=experiments/libimb_xr.so,cur=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/ab_al.txt 2>&1
cat gpurun_out/ab_al.txt
timeout 900 python tools/parity_margin.py --configs c4 > gpurun_out/margin_al.txt 2>&1; cat gpurun_out/margin_al.txt
