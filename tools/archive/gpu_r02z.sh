#!/bin/bash
# full GPU suite + smoke on the session-3 build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke_z.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_pytest_z.log 2>&1; echo pytest=$?; tail -2 gpurun_out/gpu_pytest_z.log
