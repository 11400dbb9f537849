#!/bin/bash
# A/B: per-pixel words kernel, round-1 code (FIZI_SLOW_V=1) vs SWAR + item prefetch
mkdir -p gpurun_out
out=gpurun_out/slow_ab.log; : > $out
timeout 900 python -m pytest tests -x -q -m gpu -k "c2 or c4 or cube or regime or tall or inverted or gaps or parity" >> $out 2>&1
echo "pytest rc=$?" >> $out
for v in 1 2; do
  for cfg in 4 2 3; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== V=$v C$cfg" >> $out
    FIZI_SLOW_V=$v timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items() if v})" >> $out 2>&1
  done
done
