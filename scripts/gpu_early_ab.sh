#!/bin/bash
# A/B: persistent fused kernel claims its next item and starts that item's ring
# before the current item's bookkeeping (FIZI_EARLY_NEXT=1, default) or not (=0)
mkdir -p gpurun_out
out=gpurun_out/early_ab.log; : > $out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider >> $out 2>&1
echo "pytest rc=$?" >> $out
for rep in 1 2; do
for v in 0 1; do
  for cfg in 3 4 2; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== early=$v C$cfg" >> $out
    FIZI_EARLY_NEXT=$v timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1), 'seg_joined', round(d['roofline']['stage_ms_per_step']['segment']*1e3,1), 'spot', (d.get('spot_check') or {}).get('all_match'))" >> $out 2>&1
  done
  echo "== early=$v C3 driver" >> $out
  FIZI_EARLY_NEXT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
done
done
