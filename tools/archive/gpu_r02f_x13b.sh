#!/bin/bash
# three psi^(1) slots + rotating slot reference: parity subset, then A/B against the four-slot build.
mkdir -p gpurun_out/x13
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/x13/pytest_b.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/x13/pytest_b.txt
timeout 1200 python tools/ab.py --configs c4,c5d,c2,c1 --reps 3 --steps 20 \
  --libs x4=experiments/libimb_x4.so,x3r=paper_1507_01265_b200/libimb_b200.so > gpurun_out/x13/ab_b.txt 2>&1
cat gpurun_out/x13/ab_b.txt
