#!/bin/bash
# TMWB (z-velocities + older betas in TMEM) A/B and parity.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_g.log
python tools/ab.py --configs c4,c5d,c2 --reps 3 --libs base=experiments/libimb_base.so,tmwb=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_g.txt 2>&1
cat gpurun_out/ab_g.txt
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_g.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_g.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_g.log 2>&1; echo launches=$?
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4_r02g $P > gpurun_out/ncu_full_g.log 2>&1; echo full=$?
