#!/bin/bash
# New defaults (FLUXST/BCLAMP/LFSIGN/KSHARE): config table, C4 100-step margin, C5 margins, fp32 bit identity.
mkdir -p gpurun_out/nd
bash tools/config_table.sh > gpurun_out/nd/configs.txt 2>&1; cat gpurun_out/nd/configs.txt
timeout 300 python tools/fp32_check.py > gpurun_out/nd/fp32_check.txt 2>&1; tail -7 gpurun_out/nd/fp32_check.txt
timeout 1500 python tools/parity_margin.py --configs c1,c2,c4,c4s --out gpurun_out/nd/margins.jsonl 2>&1 | cut -c1-460
timeout 1500 python tools/parity_margin.py --configs c5d,c5s --steps 30 --out gpurun_out/nd/margins.jsonl 2>&1 | cut -c1-460
