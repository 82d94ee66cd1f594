#!/bin/bash
# Full GPU suite (no -x) + default bench line + reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_f.log 2>&1; echo pytest=$? | tee -a gpurun_out/pytest_f.log
tail -40 gpurun_out/pytest_f.log
python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo bench=$?
cat gpurun_out/bench_f.json; tail -3 gpurun_out/bench_f.err
