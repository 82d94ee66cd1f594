#!/bin/bash
# limiter stores limited fluxes (IMB_FLUXST) on top of IMB_KSHARE=2: parity margins, then A/B timing.
mkdir -p gpurun_out/fx
for v in fx; do
  echo "== $v"; IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python tools/parity_margin.py --configs c1,c2,c4s --steps 20 2>&1 | tail -3
  IMB_LIB=$PWD/experiments/libimb_$v.so timeout 300 python tools/fp32_check.py 2>&1 | tail -8
done > gpurun_out/fx/parity.txt 2>&1
timeout 1200 python tools/ab.py --configs c4,c5d,c2 --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,ks2=experiments/libimb_ks2.so,fx=experiments/libimb_fx.so \
  > gpurun_out/fx/ab.txt 2>&1
timeout 600 python tools/ab.py --fp32 --configs c4,c5s --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,fx=experiments/libimb_fx.so \
  > gpurun_out/fx/ab32.txt 2>&1
cat gpurun_out/fx/parity.txt gpurun_out/fx/ab.txt gpurun_out/fx/ab32.txt
