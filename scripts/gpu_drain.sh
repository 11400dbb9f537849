#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['host_enqueue_ms_per_step'], d['host_step_gaps'], d['clocks'])" >> gpurun_out/drain_bench.log
done
