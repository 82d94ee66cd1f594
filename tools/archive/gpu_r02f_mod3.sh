#!/bin/bash
mkdir -p gpurun_out/mod3
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or config or scheme" 2>&1 | tail -1
timeout 1500 python tools/ab.py --configs c4,c5d,c2 --reps 3 --steps 20 --libs base=paper_1507_01265_b200/libimb_b200.so,mod3u=experiments/libimb_mod3u.so > gpurun_out/mod3/ab.txt 2>&1
timeout 1500 python tools/ab.py --fp32 --configs c4,c5s --reps 3 --steps 20 --libs base=paper_1507_01265_b200/libimb_b200.so,mod3u=experiments/libimb_mod3u.so >> gpurun_out/mod3/ab.txt 2>&1
cat gpurun_out/mod3/ab.txt
