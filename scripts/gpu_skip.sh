#!/bin/bash
# Diagnostics: pipeline rate with a stage skipped (upper bound of speeding it up)
mkdir -p gpurun_out
out=gpurun_out/skip.log; : > $out
for sk in none slow morph slow,morph; do
  for cfg in 4 3 2; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== skip=$sk C$cfg" >> $out
    FIZI_DIAG_SKIP=$sk timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1))" >> $out 2>&1
  done
done
