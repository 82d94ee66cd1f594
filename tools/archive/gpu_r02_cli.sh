#!/bin/bash
# FPM loop with the production halo path: speed functions
# measured on a ring of slabs pushing halos into each other (p slabs sharing
# the one GPU: a labelled stand-in), then the Table 1/2 validation as the real
# lockstep decomposition. C4 grid 1024x512x128 fp64 IORD=2 limiter.
mkdir -p gpurun_out/cli_r02_p2 gpurun_out/cli_r02_p4
C="python -m paper_1507_01265_b200.cli"
$C measure --x 448:576:16 --m 512 --l 128 --halo ring --devices 0,0 --steps 10 --max-reps 12 --out-dir gpurun_out/cli_r02_p2 > gpurun_out/cli_r02_p2/measure.log 2>&1; echo m2=$?
$C validate gpurun_out/cli_r02_p2/speed_avg.csv --total 1024 --p 2 --offsets 0,16,32,48,64 --devices 0,0 --l 128 --steps 10 --out-dir gpurun_out/cli_r02_p2 > gpurun_out/cli_r02_p2/validate.log 2>&1; echo v2=$?
$C partition gpurun_out/cli_r02_p2/speed_avg.csv --total 1024 --p 2 --out-dir gpurun_out/cli_r02_p2 > gpurun_out/cli_r02_p2/partition.log 2>&1; echo p2=$?
$C measure --x 192:320:16 --m 512 --l 128 --halo ring --devices 0,0,0,0 --steps 10 --max-reps 12 --out-dir gpurun_out/cli_r02_p4 > gpurun_out/cli_r02_p4/measure.log 2>&1; echo m4=$?
$C validate gpurun_out/cli_r02_p4/speed_avg.csv --total 1024 --p 4 --offsets 0,16,32,48,64 --devices 0,0,0,0 --l 128 --steps 10 --out-dir gpurun_out/cli_r02_p4 > gpurun_out/cli_r02_p4/validate.log 2>&1; echo v4=$?
$C partition gpurun_out/cli_r02_p4/speed_avg.csv --total 1024 --p 4 --out-dir gpurun_out/cli_r02_p4 > gpurun_out/cli_r02_p4/partition.log 2>&1; echo p4=$?
tail -8 gpurun_out/cli_r02_p2/*.log gpurun_out/cli_r02_p4/*.log
