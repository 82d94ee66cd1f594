#!/bin/bash
# full GPU suite + smoke + C5 numbers on the per-mode XR build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_aq.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_pytest_aq.log 2>&1; echo pytest=$?; tail -1 gpurun_out/gpu_pytest_aq.log
bash tools/config_table.sh > gpurun_out/configs_aq.txt 2>&1; cat gpurun_out/configs_aq.txt
P="python tools/profile_step.py --config c5d --warm 1 --steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/fused_c5d_r02aq $P > gpurun_out/ncu_c5d_aq.log 2>&1; echo c5d=$?
