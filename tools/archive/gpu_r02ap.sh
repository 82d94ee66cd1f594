#!/bin/bash
# which IORD=3 passes keep the extra rows: all (xr3), MODE 0+2 (xm5), MODE 0 only (xm1)
mkdir -p gpurun_out
for v in xm5 xm1; do IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "iord3 or scheme" > gpurun_out/pytest_ap_$v.log 2>&1; echo $v pytest=$?; tail -1 gpurun_out/pytest_ap_$v.log; done
python tools/ab.py --configs c5d --reps 3 --libs xr3=experiments/libimb_xr3.so,xm5=experiments/libimb_xm5.so,xm1=experiments/libimb_xm1.so > gpurun_out/ab_ap.txt 2>&1
python tools/ab.py --fp32 --configs c5s --reps 3 --libs xr3=experiments/libimb_xr3.so,xm5=experiments/libimb_xm5.so,xm1=experiments/libimb_xm1.so >> gpurun_out/ab_ap.txt 2>&1
cat gpurun_out/ab_ap.txt
