#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/slowgrid.log; : > $out
for g in 8 5 3 16 32; do
  for cfg in 4 2 3; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== grid=$g/SM C$cfg" >> $out
    FIZI_SLOW_GRID=$g timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'slow', round(d['roofline']['stage_ms_per_step']['slow']*1e3,1))" >> $out 2>&1
  done
done
