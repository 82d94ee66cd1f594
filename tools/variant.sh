#!/bin/bash
# Build an A/B variant of the library: tools/variant.sh NAME "NVCC flags"
#   -> experiments/libimb_NAME.so (git-ignored; travels to the GPU box)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=/tmp/imb_var_$1
make -s -C $ROOT/paper_1507_01265_b200/csrc BUILD=$B OUT=$ROOT/experiments/libimb_$1.so NVEXTRA="$2" -j8
