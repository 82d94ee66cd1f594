#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused or config or group or matrix" > gpurun_out/pytest_ab2.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_ab2.log
python tools/ab.py --configs c4,c5d --reps 3 --libs tms=paper_1507_01265_b200/libimb_b200.so,notms=experiments/libimb_notms.so > gpurun_out/ab2.txt 2>&1
cat gpurun_out/ab2.txt
