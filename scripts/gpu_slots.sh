#!/bin/bash
# A/B: call slots (pipelined calls in flight) 4 / 6 / 8 on C3, C4, C2
mkdir -p gpurun_out
out=gpurun_out/slots.log; : > $out
for lib in libfizi.so libfizi_s6.so libfizi_s8.so; do
  for cfg in 3 4 2; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== $lib C$cfg" >> $out
    FIZI_LIB=$lib timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
  done
  echo "== $lib C3 driver" >> $out
  FIZI_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
done
