#!/bin/bash
# Quick GPU iteration: parity tests (fused subset) + per-config step timing.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or config or group or step_host" > gpurun_out/pytest_quick.log 2>&1
echo "pytest=$?"; tail -3 gpurun_out/pytest_quick.log
for c in c4 c2 c1 c5d; do python tools/profile_step.py --config $c --warm 2 --steps 10; done
python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10
