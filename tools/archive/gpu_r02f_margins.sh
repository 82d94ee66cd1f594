#!/bin/bash
# final-kernel parity margins: C4 fp64 100 steps on four seeds, C5 fp64/fp32 100 steps, C4 fp32
mkdir -p gpurun_out/margins
timeout 1200 python tools/parity_margin.py --configs c4 --seeds 42,7,123,2024 --out gpurun_out/margins/final.jsonl 2>&1 | cut -c1-300
timeout 2400 python tools/parity_margin.py --configs c1,c2,c4s,c5d,c5s --out gpurun_out/margins/final.jsonl 2>&1 | cut -c1-300
