#!/bin/bash
# final-layout refresh: bench line, reference arm, config table, launch list, ncu of C4 fp64
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_ao.json 2> gpurun_out/bench_ao.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref_ao.json 2> gpurun_out/bench_ref_ao.err; echo ref=$?
bash tools/config_table.sh > gpurun_out/configs_ao.txt 2>&1; cat gpurun_out/configs_ao.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ao.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_ao.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4d_r02ao python tools/profile_step.py --config c4 --warm 1 --steps 1 > gpurun_out/ncu_c4d_ao.log 2>&1; echo c4d=$?
P="python tools/profile_step.py --config c5d --warm 1 --steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/fused_c5d_r02ao $P > gpurun_out/ncu_c5d_ao.log 2>&1; echo c5d=$?
