#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/fold2.log; : > $out
timeout 1200 python -m pytest tests -x -q -m gpu -k "config or pipelined or relearn or track or c2 or c4 or 4x4 or generic" -p no:cacheprovider >> $out 2>&1
echo "pytest rc=$?" >> $out
TL_CONFIG=3 TL_WARM=5 TL_NCALLS=20 timeout 300 python scripts/timeline.py > gpurun_out/tl_fold2.log 2>&1
for cfg in 3 4 2; do
  st=100; [ $cfg = 4 ] && st=40
  echo "== C$cfg" >> $out
  timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'ccl', round(d['roofline']['stage_ms_per_step']['ccl']*1e3,1), 'spot', (d.get('spot_check') or {}).get('all_match'))" >> $out 2>&1
done
echo "== C3 driver" >> $out
for i in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
done
