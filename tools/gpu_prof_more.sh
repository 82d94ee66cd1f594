#!/bin/bash
# Extra ncu evidence: the fp32 C4 step kernel and both IORD=3 launches on the C5 grid.
mkdir -p gpurun_out
P32="python tools/profile_step.py --config c4 --fp32 --warm 1 --steps 1"
$P32 > gpurun_out/p32.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4_fp32 $P32 > gpurun_out/ncu32.log 2>&1; echo fp32=$?
P5="python tools/profile_step.py --config c5d --warm 1 --steps 1"
$P5 > gpurun_out/p5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/fused_c5_fp64 $P5 > gpurun_out/ncu5.log 2>&1; echo c5=$?
