#!/bin/bash
mkdir -p gpurun_out/cs
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "iord3 or scheme or config" 2>&1 | tail -2
timeout 1500 python tools/ab.py --configs c5d --reps 3 --steps 10 --libs nocs=experiments/libimb_nocs.so,cs=paper_1507_01265_b200/libimb_b200.so > gpurun_out/cs/ab.txt 2>&1
timeout 1500 python tools/ab.py --fp32 --configs c5s --reps 3 --steps 10 --libs nocs=experiments/libimb_nocs.so,cs=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/cs/ab.txt 2>&1
cat gpurun_out/cs/ab.txt
