#!/bin/bash
# host-step pipeline: ramped chunks (default) vs uniform 16; and the bit-identity test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "step_host" > gpurun_out/pytest_aa.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_aa.log
for r in 1 2 3; do
  for c in 0 16; do
    IMB_PIPE_CHUNKS=$c python bench.py --steps 5 --warmup 3 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks $c', round(d['e2e']['value'],3))"
  done
done 2>&1 | tee gpurun_out/e2e_ramp.txt
