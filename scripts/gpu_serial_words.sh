#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/serial_words.log; : > $out
for v in 0 1; do
  for cfg in 4 2 3 5; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== serial_words=$v C$cfg" >> $out
    FIZI_SERIAL_WORDS=$v timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
  done
done
