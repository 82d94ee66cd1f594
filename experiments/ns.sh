#!/bin/bash
# fp64 lane-vector shapes: NS=2 x K=2 (product), NS=1 x K=4 (v10, v11 with the star carry), NS=4 x K=1 (v12).
export IMB_LIB=$PWD/experiments/libimb_variants.so
for v in 0 10 11 12; do echo -n "v$v c4: "; IMB_RWV=$v python tools/profile_step.py --config c4 --warm 3 --steps 20 | sed 's/.*-> //'; done
