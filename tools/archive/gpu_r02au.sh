#!/bin/bash
# C5 fp64: pass 2 (MODE 1) with the extra rows and shorter segments (IMB_SEG_MAX)
mkdir -p gpurun_out
for seg in 0 512 256 128; do
  for lib in paper_1507_01265_b200/libimb_b200.so experiments/libimb_xm7.so; do
    if [ $seg = 0 ]; then unset IMB_SEG_MAX; else export IMB_SEG_MAX=$seg; fi
    r=$(IMB_LIB=$PWD/$lib python tools/profile_step.py --config c5d --warm 3 --steps 10 | grep -oE "[0-9.]+ Gcell/s")
    echo "seg_max=$seg $(basename $lib): $r"
  done
done 2>&1 | tee gpurun_out/c5_segmax.txt
