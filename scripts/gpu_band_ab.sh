#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/band_ab.log; : > $out
FIZI_LIB=libfizi_br32.so timeout 900 python -m pytest tests -x -q -m gpu -k "exhaustive or config4 or pipelined_c4 or config3 or 5x5" -p no:cacheprovider >> $out 2>&1
echo "pytest br32 rc=$?" >> $out
for lib in libfizi.so libfizi_br24.so libfizi_br32.so; do
  for cfg in 4 3 2; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== $lib C$cfg" >> $out
    FIZI_LIB=$lib timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'morph', round(d['roofline']['stage_ms_per_step']['morph']*1e3,1))" >> $out 2>&1
  done
done
