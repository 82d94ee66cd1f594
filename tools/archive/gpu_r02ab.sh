#!/bin/bash
# host-step pipeline chunking sweep (uniform counts, ramp bases), e2e only
mkdir -p gpurun_out
run() { python bench.py --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['e2e']['value'],3))"; }
for r in 1 2; do
  for c in 12 16 20 24 32; do IMB_PIPE_CHUNKS=$c run "uniform $c"; done
  for b in 8 16 32; do IMB_PIPE_BASE=$b run "ramp base $b"; done
done 2>&1 | tee gpurun_out/e2e_sweep.txt
