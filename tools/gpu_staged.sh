#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_full.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_full.log
for c in c5d c5s; do python tools/profile_step.py --config $c --warm 1 --steps 3; done
