#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (SURVEY.md §4 item 5). One line per (tool, case): exit code and the summary.
# Note: the round-1 GPU pool refuses compute-sanitizer (it has left GPUs needing a
# reset there); tools/checked_build.sh + tests/test_checked.py stand in for it.
# Kept for machines where the sanitizer is allowed.
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for c in ${CASES:-fused_f64 fused_f32 fused_plain fused_iord3 fused_l64 fused_l32 staged group group_flags}; do
    t0=$(date +%s)
    timeout ${TMO:-600} $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $c > gpurun_out/san_${tool}_$c.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(( $(date +%s) - t0 ))s: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_$c.log | tail -1)"
  done
done
