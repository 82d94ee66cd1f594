#!/bin/bash
# extra y-face in four (segment, element) pieces on one warp per scheduler (IMB_XR_YWARP=3): parity, A/B
mkdir -p gpurun_out/y4
for v in y4a; do IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or config or extra or xr" 2>&1 | tail -2; done > gpurun_out/y4/parity.txt 2>&1
cat gpurun_out/y4/parity.txt
timeout 1500 python tools/ab.py --configs c4 --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,y4a=experiments/libimb_y4a.so,y4b=experiments/libimb_y4b.so,y4c=experiments/libimb_y4c.so > gpurun_out/y4/ab.txt 2>&1
cat gpurun_out/y4/ab.txt
