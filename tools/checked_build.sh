#!/bin/bash
# Checked build: libimb_b200_checked.so with the device-side bounds asserts of
# -DIMB_CHECKED (plane indices, rows, shared-memory offsets, halo-push planes).
# compute-sanitizer is not available on this GPU pool; this build plus the
# small cases of tools/sanitize_cases.py and the parity suite stand in for it:
#   IMB_LIB=$PWD/paper_1507_01265_b200/libimb_b200_checked.so python tools/sanitize_cases.py
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -j"$(nproc)" -C "$ROOT/paper_1507_01265_b200/csrc" BUILD="$ROOT/paper_1507_01265_b200/build/checked" \
  OUT="$ROOT/paper_1507_01265_b200/libimb_b200_checked.so" NVEXTRA="-DIMB_CHECKED"
