#!/bin/bash
# k-pair shared extrema (IMB_KSHARE bits): parity margin on c2 (50 steps), then A/B timing.
mkdir -p gpurun_out/ks
for v in ks1 ks2 ks3; do
  echo "== $v"; IMB_LIB=$PWD/experiments/libimb_$v.so timeout 300 python tools/parity_margin.py --configs c1,c2 2>&1 | tail -2
done > gpurun_out/ks/parity.txt 2>&1
timeout 1200 python tools/ab.py --configs c4,c5d --reps 3 --steps 20 \
  --libs base=paper_1507_01265_b200/libimb_b200.so,ks1=experiments/libimb_ks1.so,ks2=experiments/libimb_ks2.so,ks3=experiments/libimb_ks3.so \
  > gpurun_out/ks/ab.txt 2>&1
cat gpurun_out/ks/parity.txt gpurun_out/ks/ab.txt
