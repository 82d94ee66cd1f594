#!/bin/bash
# three psi^(1) slots with the early donor (IMB_X1_3, needs FLUXST): parity subset, then A/B against four slots.
mkdir -p gpurun_out/x13
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or config or group or step_host or xr or extra or scheme" > gpurun_out/x13/pytest.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/x13/pytest.txt
timeout 600 python tools/parity_margin.py --configs c2,c4 --steps 20 2>&1 | cut -c1-400 > gpurun_out/x13/margins.txt; cat gpurun_out/x13/margins.txt
timeout 1200 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs x4=experiments/libimb_x4.so,x3=paper_1507_01265_b200/libimb_b200.so > gpurun_out/x13/ab.txt 2>&1
cat gpurun_out/x13/ab.txt
