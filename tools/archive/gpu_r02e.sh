#!/bin/bash
# Round-2 state check after the session restart: GPU suite, bench line,
# per-config table, launch list of the bench command, one full ncu capture.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; nvidia-smi >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_e.log 2>&1; echo pytest=$? | tee -a gpurun_out/pytest_e.log
tail -25 gpurun_out/pytest_e.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo bench=$?
cat gpurun_out/bench_e.json; tail -5 gpurun_out/bench_e.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_e.json 2> gpurun_out/bench_ref_e.err; echo ref=$?
cat gpurun_out/bench_ref_e.json
for c in c4 c2 c5d c5s; do python tools/profile_step.py --config $c --warm 2 --steps 10; done > gpurun_out/configs_e.txt 2>&1
python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10 >> gpurun_out/configs_e.txt 2>&1
cat gpurun_out/configs_e.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_e.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_e.log 2>&1; echo launches=$?
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4_r02e $P > gpurun_out/ncu_full_e.log 2>&1; echo full=$?
P="python tools/profile_step.py --config c5d --warm 1 --steps 1"
ncu --set full --clock-control none -k regex:k_fused -s 3 -c 3 -o gpurun_out/fused_c5d_r02e $P > gpurun_out/ncu_full_e5.log 2>&1; echo full5=$?
