#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_ab4.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ab4.log
python tools/ab.py --configs c4,c5d --reps 4 --libs cache=paper_1507_01265_b200/libimb_b200.so,staronly=experiments/libimb_staronly.so,notms=experiments/libimb_notms.so > gpurun_out/ab4.txt 2>&1
cat gpurun_out/ab4.txt
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4_r02d $P > gpurun_out/ncu_full_d.log 2>&1; echo full=$?
