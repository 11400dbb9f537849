#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/c5grid.log; : > $out
for rep in 1 2; do for g in 8 16; do
  echo "== grid=$g C5" >> $out
  FIZI_SLOW_GRID=$g timeout 300 python bench.py --config 5 --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'slow', round(d['roofline']['stage_ms_per_step']['slow']*1e3,1))" >> $out 2>&1
done; done
