#!/bin/bash
# Build libimb_b200.so from a git revision (default HEAD) into experiments/libimb_<name>.so,
# for A/B runs against the working tree with IMB_LIB (see abn.sh).
#   experiments/build_lib.sh base [REV] [extra nvcc flags...]
set -e
name=${1:?name}; rev=${2:-HEAD}; shift 2 || shift 1
ROOT=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$ROOT" archive "$rev" paper_1507_01265_b200/csrc paper_1507_01265_b200/include include | tar -x -C "$tmp"
make -s -j8 -C "$tmp/paper_1507_01265_b200/csrc" BUILD="$tmp/build" OUT="$ROOT/experiments/libimb_$name.so" NVEXTRA="$*"
rm -rf "$tmp"
echo "built experiments/libimb_$name.so from $rev"
