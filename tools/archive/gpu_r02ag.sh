#!/bin/bash
# XR variants: extra y-face split over warps 0/15 (cur) vs on warp 15 (xr) vs pre-XR (head)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused or config or scheme" > gpurun_out/pytest_ag.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ag.log
python tools/ab.py --configs c4,c5d --reps 3 --libs head=experiments/libimb_head.so,xr=experiments/libimb_xr.so,split=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_ag.txt 2>&1
cat gpurun_out/ab_ag.txt
