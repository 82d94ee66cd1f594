#!/bin/bash
mkdir -p gpurun_out
python tools/fp32_check.py > gpurun_out/fp32_check.txt 2>&1; echo fp32check=$?
cat gpurun_out/fp32_check.txt
for c in c4 c5s; do python tools/profile_step.py --config $c --warm 2 --steps 10; done > gpurun_out/configs_b.txt 2>&1
python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10 >> gpurun_out/configs_b.txt 2>&1
cat gpurun_out/configs_b.txt
python tools/parity_margin.py --configs c5s,c4s,c5d --out gpurun_out/margins_b.jsonl > gpurun_out/margins_b.log 2>&1; echo margins=$?
cat gpurun_out/margins_b.log
