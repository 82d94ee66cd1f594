#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_i.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_i.log
python tools/ab.py --configs c4,c5d --reps 3 --libs tmwb1=experiments/libimb_tmwb1.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_i.txt 2>&1
cat gpurun_out/ab_i.txt
for pf in 0 2; do IMB_PF=$pf python tools/profile_step.py --config c4 --warm 3 --steps 20; done
