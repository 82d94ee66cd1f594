#!/bin/bash
# Full verification on one B200: GPU suite, smoke, per-config table, bench line
# (own arm + reference arm). Output under gpurun_out/verify/.
O=gpurun_out/verify; mkdir -p $O
timeout 1500 python -m pytest tests/ -x -q -m gpu > $O/gpu_pytest.txt 2>&1; echo pytest=$?; tail -3 $O/gpu_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo smoke=$?
bash tools/config_table.sh > $O/configs.txt 2>&1; echo configs=$?; cat $O/configs.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?; cat $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?; cat $O/bench_ref.json
