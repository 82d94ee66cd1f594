#!/bin/bash
# session-3 refresh: config table, default bench line, reference arm
mkdir -p gpurun_out
bash tools/config_table.sh > gpurun_out/configs_x.txt 2>&1
python bench.py > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err
python bench.py --impl reference > gpurun_out/bench_ref_x.json 2> gpurun_out/bench_ref_x.err
cat gpurun_out/configs_x.txt gpurun_out/bench_x.json gpurun_out/bench_ref_x.json
