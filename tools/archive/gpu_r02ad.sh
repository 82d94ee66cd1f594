#!/bin/bash
# fp64 7-point extrema sharing first-level compares: A/B + parity (incl. full-size C4/C5)
mkdir -p gpurun_out
python tools/ab.py --configs c4,c5d --reps 3 --libs head=experiments/libimb_head.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_ad.txt 2>&1
cat gpurun_out/ab_ad.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_ad.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ad.log
