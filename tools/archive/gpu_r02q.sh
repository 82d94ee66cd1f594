#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
python tools/ab.py --configs c4,c5d,c2 --reps 3 --libs noyoff=experiments/libimb_noyoff.so,yoff=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_q.txt 2>&1
cat gpurun_out/ab_q.txt
