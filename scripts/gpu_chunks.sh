#!/bin/bash
# per-pixel stage over chunk items with a per-warp TMA ring: GPU suite + bench lines
mkdir -p gpurun_out
out=gpurun_out/chunks.log; : > $out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider >> $out 2>&1
echo "pytest rc=$?" >> $out
for cfg in 4 2 3 5; do
  st=100; [ $cfg = 4 ] && st=40
  echo "== C$cfg" >> $out
  timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items() if v}, 'spot', (d.get('spot_check') or {}).get('all_match'))" >> $out 2>&1
done
for n in 2 6 8; do
  echo "== FIZI_SLOW_CTAS=$n C4 / C2" >> $out
  for cfg in 4 2; do
  st=100; [ $cfg = 4 ] && st=40
  FIZI_SLOW_CTAS=$n timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'slow', round(d['roofline']['stage_ms_per_step']['slow']*1e3,1))" >> $out 2>&1
  done
done
echo "== C3 driver" >> $out
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
