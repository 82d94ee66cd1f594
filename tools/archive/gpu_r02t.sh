#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_checked.py -x -q -p no:cacheprovider > gpurun_out/pytest_t.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_t.log
timeout 600 python -m pytest tests/test_multiproc_gpu.py -x -q -p no:cacheprovider -k "ipc_ring" > gpurun_out/pytest_t_mp.log 2>&1; echo mp=$?; tail -1 gpurun_out/pytest_t_mp.log
python tools/ab.py --configs c4,c5d,c2 --reps 3 --libs head=experiments/libimb_head.so,cur=paper_1507_01265_b200/libimb_b200.so > gpurun_out/ab_t.txt 2>&1
python tools/ab.py --fp32 --configs c4,c5s --reps 2 --libs head=experiments/libimb_head.so,cur=paper_1507_01265_b200/libimb_b200.so >> gpurun_out/ab_t.txt 2>&1
cat gpurun_out/ab_t.txt
