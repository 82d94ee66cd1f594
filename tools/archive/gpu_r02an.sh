#!/bin/bash
# IORD=3 passes with the split extra y-face: MODE 1 (sm3) or MODE 2 (sm5) as well
mkdir -p gpurun_out
for v in sm3 sm5; do IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "iord3 or scheme" > gpurun_out/pytest_an_$v.log 2>&1; echo $v pytest=$?; tail -1 gpurun_out/pytest_an_$v.log; done
python tools/ab.py --configs c5d --reps 3 --libs cur=paper_1507_01265_b200/libimb_b200.so,sm3=experiments/libimb_sm3.so,sm5=experiments/libimb_sm5.so > gpurun_out/ab_an.txt 2>&1
cat gpurun_out/ab_an.txt
