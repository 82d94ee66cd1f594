#!/bin/bash
# fp32 packed pairs (FADD2/FMUL2/FFMA2): bit-exact parity + A/B against the previous head
mkdir -p gpurun_out
./experiments/micro/p2check
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_u.log 2>&1; echo fp32_check=$?; cat gpurun_out/fp32_check_u.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_u.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_u.log
python tools/ab.py --fp32 --configs c4,c5s --reps 3 --libs head=experiments/libimb_head.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_u.txt 2>&1

cat gpurun_out/ab_u.txt
