#!/bin/bash
# XR build: full GPU suite, bench line, config table, ncu of the C4 step (fp64, fp32)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_pytest_ah.log 2>&1; echo pytest=$?; tail -1 gpurun_out/gpu_pytest_ah.log
python bench.py > gpurun_out/bench_ah.json 2> gpurun_out/bench_ah.err; echo bench=$?
bash tools/config_table.sh > gpurun_out/configs_ah.txt 2>&1; cat gpurun_out/configs_ah.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ah.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_ah.log 2>&1; echo launches=$?
for spec in "c4:c4d:" "c4 --fp32:c4s:"; do
  IFS=: read args tag x <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_${tag}_r02ah python tools/profile_step.py --config $args --warm 1 --steps 1 > gpurun_out/ncu_${tag}_ah.log 2>&1; echo $tag=$?
done
