mkdir -p gpurun_out/p1
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
$P > gpurun_out/p1/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/p1/fused_c4 $P > gpurun_out/p1/ncu_full.log 2>&1; echo full=$?
ncu -i gpurun_out/p1/fused_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/p1/c4_sass.csv 2>/dev/null; echo $?
ncu -i gpurun_out/p1/fused_c4.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/p1/c4_src.csv 2>/dev/null; echo $?
ls -la gpurun_out/p1
