#!/bin/bash
# A/B: labelling stage on the morphology's stream (FIZI_MERGE_MC=1)
mkdir -p gpurun_out
out=gpurun_out/merge_ab.log; : > $out
for m in 0 1; do
  if [ $m = 1 ]; then export FIZI_MERGE_MC=1; else unset FIZI_MERGE_MC; fi
  TL_CONFIG=3 TL_WARM=5 TL_NCALLS=20 timeout 300 python scripts/timeline.py > gpurun_out/tl_merge_$m.log 2>&1
  for cfg in 3 4 2 5; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== merge=$m C$cfg" >> $out
    timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
  done
  echo "== merge=$m C3 driver" >> $out
  for i in 1 2 3; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
  done
done
