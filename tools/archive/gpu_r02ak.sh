#!/bin/bash
# who computes the extra row's y-face: warp 15 (cur), warp 0 (yw0), one segment each (yw2)
mkdir -p gpurun_out
for v in yw0 yw2; do
  IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused or config or scheme" > gpurun_out/pytest_ak_$v.log 2>&1; echo $v pytest=$?; tail -1 gpurun_out/pytest_ak_$v.log
  IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python tools/fp32_check.py 2>&1 | tail -2
done
python tools/ab.py --configs c4,c5d --reps 3 --libs xr=experiments/libimb_xr.so,cur=paper_1507_01265_b200/libimb_b200.so,yw0=experiments/libimb_yw0.so,yw2=experiments/libimb_yw2.so > gpurun_out/ab_ak.txt 2>&1
python tools/ab.py --fp32 --configs c4,c5s --reps 2 --libs xr=experiments/libimb_xr.so,cur=paper_1507_01265_b200/libimb_b200.so,yw0=experiments/libimb_yw0.so >> gpurun_out/ab_ak.txt 2>&1
cat gpurun_out/ab_ak.txt
