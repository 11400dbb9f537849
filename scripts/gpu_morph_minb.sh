#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/morph_minb.log; : > $out
for lib in libfizi.so libfizi_mm5.so libfizi_mm6.so libfizi_mm8.so; do
  for cfg in 4 3; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== $lib C$cfg" >> $out
    FIZI_LIB=$lib timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'morph', round(d['roofline']['stage_ms_per_step']['morph']*1e3,1))" >> $out 2>&1
  done
done
