#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_c.log
python tools/fp32_check.py > gpurun_out/fp32_check_c.txt 2>&1; cat gpurun_out/fp32_check_c.txt
for c in c4 c2 c5d c5s; do python tools/profile_step.py --config $c --warm 2 --steps 10; done > gpurun_out/configs_c.txt 2>&1
python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10 >> gpurun_out/configs_c.txt 2>&1
cat gpurun_out/configs_c.txt
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4_r02c $P > gpurun_out/ncu_full_c.log 2>&1; echo full=$?
