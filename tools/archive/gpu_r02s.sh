#!/bin/bash
# Linear (tile, plane) split vs the grid split (env IMB_LIN), parity under both.
mkdir -p gpurun_out
for lin in 1 0; do
  IMB_LIN=$lin timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_s$lin.log 2>&1; echo pytest_lin$lin=$?; tail -1 gpurun_out/pytest_s$lin.log
done
IMB_LIN=1 timeout 600 python -m pytest tests/test_multiproc_gpu.py -x -q -p no:cacheprovider -k "ipc_ring" > gpurun_out/pytest_s_mp.log 2>&1; echo mp=$?; tail -1 gpurun_out/pytest_s_mp.log
for rep in 1 2 3; do for cfg in "c4" "c5d" "c2" "c4 --fp32" "c5s --fp32" "c1"; do for lin in 0 1; do
  echo -n "lin=$lin $cfg: "; IMB_LIN=$lin python tools/profile_step.py --config $cfg --warm 3 --steps 20 | sed 's/.*-> //'
done; done; done > gpurun_out/lin_s.txt 2>&1
sort gpurun_out/lin_s.txt
