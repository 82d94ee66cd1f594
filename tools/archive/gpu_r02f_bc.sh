#!/bin/bash
# beta pre-clamp (IMB_BCLAMP) and shared limit/flux sign test (IMB_LFSIGN) on top of fx: parity, then A/B.
mkdir -p gpurun_out/bc
for v in bc lf; do
  echo "== $v"; IMB_LIB=$PWD/experiments/libimb_$v.so timeout 600 python tools/parity_margin.py --configs c1,c2 2>&1 | tail -2 | cut -c1-420
  IMB_LIB=$PWD/experiments/libimb_$v.so timeout 300 python tools/fp32_check.py 2>&1 | tail -6
done > gpurun_out/bc/parity.txt 2>&1
timeout 1200 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,fx=experiments/libimb_fx.so,bc=experiments/libimb_bc.so,lf=experiments/libimb_lf.so \
  > gpurun_out/bc/ab.txt 2>&1
timeout 600 python tools/ab.py --fp32 --configs c4,c5s --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,fx=experiments/libimb_fx.so,bc=experiments/libimb_bc.so,lf=experiments/libimb_lf.so \
  > gpurun_out/bc/ab32.txt 2>&1
cat gpurun_out/bc/parity.txt gpurun_out/bc/ab.txt gpurun_out/bc/ab32.txt
