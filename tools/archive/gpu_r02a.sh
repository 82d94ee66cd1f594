#!/bin/bash
# Round-2 first GPU pass: the whole GPU suite (incl. full-size parity), the
# default bench line, per-config step times and one full ncu capture of the
# C4 fp64 step kernel.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo pytest=$? | tee -a gpurun_out/pytest.log
tail -3 gpurun_out/pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
for c in c4 c2 c5d c5s; do python tools/profile_step.py --config $c --warm 2 --steps 10; done > gpurun_out/configs.txt 2>&1
python tools/profile_step.py --config c4 --fp32 --warm 2 --steps 10 >> gpurun_out/configs.txt 2>&1
cat gpurun_out/configs.txt
P="python tools/profile_step.py --config c4 --warm 1 --steps 1"
$P > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_c4_r02a $P > gpurun_out/ncu_full.log 2>&1; echo full=$?
