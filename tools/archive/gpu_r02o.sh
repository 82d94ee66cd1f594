#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err; echo bench=$?; cat gpurun_out/bench_o.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_o.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_o.log 2>&1; echo launches=$?
for spec in "c4:c4d:1" "c5d:c5d:2"; do
  IFS=: read args tag cnt <<< "$spec"
  P="python tools/profile_step.py --config $args --warm 1 --steps 1"
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s $cnt -c $cnt -o gpurun_out/fused_${tag}_r02o $P > gpurun_out/ncu_${tag}_o.log 2>&1; echo $tag=$?
done
