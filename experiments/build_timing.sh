#!/bin/bash
# Debug build with per-phase cycle accounting (IMB_PHASE_TIMING) -> experiments/libimb_timing.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=/tmp/imb_timing_build
rm -rf $B && mkdir -p $B
make -s -C $ROOT/paper_1507_01265_b200/csrc BUILD=$B OUT=$ROOT/experiments/libimb_timing.so NVEXTRA="-DIMB_PHASE_TIMING" -j8
