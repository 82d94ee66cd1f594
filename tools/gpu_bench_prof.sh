#!/bin/bash
# Round evidence: bench line (default config) + ncu launch list + one full ncu capture.
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
cat gpurun_out/bench_ref.json
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4 $P > gpurun_out/ncu_full.log 2>&1; echo full=$?
