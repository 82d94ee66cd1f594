#!/bin/bash
# ncu captures of every fused instantiation the BASELINE configs run.
mkdir -p gpurun_out
for spec in "c4 --fp32:c4s:1" "c5d:c5d:2" "c5s:c5s:2" "c4:c4d:1"; do
  IFS=: read args tag cnt <<< "$spec"
  P="python tools/profile_step.py --config $args --warm 1 --steps 1"
  ncu --set full --clock-control none --import-source on -k regex:k_fused -s $cnt -c $cnt -o gpurun_out/fused_${tag}_r02j $P > gpurun_out/ncu_${tag}_j.log 2>&1; echo $tag=$?
done
