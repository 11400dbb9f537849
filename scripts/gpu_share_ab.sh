#!/bin/bash
# A/B: per-pixel words in the fused kernel shared by the CTA's warps (FIZI_INLINE=2)
mkdir -p gpurun_out
out=gpurun_out/share_ab.log; : > $out
FIZI_INLINE=2 timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider >> $out 2>&1
echo "pytest (FIZI_INLINE=2) rc=$?" >> $out
for v in 0 2; do
  for cfg in 4 2 3; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== INLINE=$v C$cfg" >> $out
    FIZI_INLINE=$v timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items() if v}, 'spot', (d.get('spot_check') or {}).get('all_match'))" >> $out 2>&1
  done
done
