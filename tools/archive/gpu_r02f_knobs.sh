#!/bin/bash
# runtime knobs re-swept on the three-slot kernel (C4 fp64): L2 prefetch distance, plan_grid warm-up weight
mkdir -p gpurun_out/knobs
{
for pf in 0 1 2 3; do echo "IMB_PF=$pf"; IMB_PF=$pf python tools/profile_step.py --config c4 --warm 3 --steps 20 | tail -1; done
for w in 2 3 4 5; do echo "IMB_WARM=$w"; IMB_WARM=$w python tools/profile_step.py --config c4 --warm 3 --steps 20 | tail -1; done
echo "IMB_GRAPH=0"; IMB_GRAPH=0 python tools/profile_step.py --config c4 --warm 3 --steps 20 | tail -1
} > gpurun_out/knobs/c4.txt 2>&1
cat gpurun_out/knobs/c4.txt
