#!/bin/bash
# r02f ncu evidence on the final kernels: C4 fp64 (with SASS page), C5 fp64, C5 fp32, bench launch list.
O=gpurun_out/r02f; mkdir -p $O
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
$P > $O/p4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o $O/fused_c4_fp64 $P > $O/ncu4.log 2>&1; echo c4=$?
ncu -i $O/fused_c4_fp64.ncu-rep --page source --csv --print-source sass > $O/c4_sass.csv 2>/dev/null
P5="python tools/profile_step.py --config c5d --warm 1 --steps 1"
$P5 > $O/p5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o $O/fused_c5_fp64 $P5 > $O/ncu5.log 2>&1; echo c5d=$?
P5s="python tools/profile_step.py --config c5s --warm 1 --steps 1"
$P5s > $O/p5s.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o $O/fused_c5_fp32 $P5s > $O/ncu5s.log 2>&1; echo c5s=$?
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo launches=$?
ls -la $O
