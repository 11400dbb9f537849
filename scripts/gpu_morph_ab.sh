#!/bin/bash
# A/B: morphology run extraction, lane-serial (round 1, -DFIZI_MORPH_SERIAL_RUNS) vs warp-parallel
mkdir -p gpurun_out
out=gpurun_out/morph_ab.log; : > $out
timeout 1200 python -m pytest tests -x -q -m gpu -k "morph or exhaust or 5x5 or 4x4 or config or c4 or tall or gaps or parity" >> $out 2>&1
echo "pytest rc=$?" >> $out
for lib in libfizi_serialruns.so libfizi.so; do
  for cfg in 4 3 2; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== $lib C$cfg" >> $out
    FIZI_LIB=$lib timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items() if v})" >> $out 2>&1
  done
  echo "== $lib C3 driver" >> $out
  FIZI_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), d['spot_check'])" >> $out 2>&1
done
