#!/bin/bash
# Experimental build with runtime-selectable fused-kernel variants -> experiments/libimb_variants.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=/tmp/imb_variants_build
rm -rf $B && mkdir -p $B
make -s -C $ROOT/paper_1507_01265_b200/csrc BUILD=$B OUT=$ROOT/experiments/libimb_variants.so NVEXTRA="-DIMB_FUSED_VARIANTS $EXTRA" -j8
