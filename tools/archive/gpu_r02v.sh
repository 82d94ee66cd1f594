#!/bin/bash
# P2 bitwise unit check; e2e pipeline chunk-count sweep
mkdir -p gpurun_out
./experiments/micro/p2check > gpurun_out/p2check.txt 2>&1; cat gpurun_out/p2check.txt
for c in 8 16 24 42; do
  for r in 1 2; do
    IMB_PIPE_CHUNKS=$c python bench.py --steps 5 --warmup 3 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks $c', round(d['e2e']['value'],3), round(d['value'],2))"
  done
done 2>&1 | tee gpurun_out/e2e_chunks.txt
