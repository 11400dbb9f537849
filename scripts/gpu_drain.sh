#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/drain_bench.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['clocks'], d['host_step_gaps']['first_us'])" >> gpurun_out/drain_bench.log
done
timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['clocks'])" >> gpurun_out/drain_bench.log
