#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "extra_row or staged" > gpurun_out/pytest_av.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_av.log
