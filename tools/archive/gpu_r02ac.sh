#!/bin/bash
# session-3 captures: launch list of the default bench, ncu --set full of C5 fp64 (both launches, MODE 2 with the bounds prefetch)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ac.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_ac.log 2>&1; echo launches=$?
P="python tools/profile_step.py --config c5d --warm 1 --steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/fused_c5d_r02ac $P > gpurun_out/ncu_c5d_ac.log 2>&1; echo c5d=$?
ls -la gpurun_out/*.ncu-rep
