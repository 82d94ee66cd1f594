#!/bin/bash
# fp64: which warp takes the second half of the extra y-face (15 = cur, or 1, 3, 5)
mkdir -p gpurun_out
IMB_LIB=$PWD/experiments/libimb_ys3.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused or config" 2>&1 | tail -1
python tools/ab.py --configs c4 --reps 3 --libs cur=paper_1507_01265_b200/libimb_b200.so,ys1=experiments/libimb_ys1.so,ys3=experiments/libimb_ys3.so,ys5=experiments/libimb_ys5.so > gpurun_out/ab_at.txt 2>&1
cat gpurun_out/ab_at.txt
