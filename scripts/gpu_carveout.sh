#!/bin/bash
# A/B: preferred shared-memory carveout of the per-call kernels (FIZI_CARVEOUT)
mkdir -p gpurun_out
out=gpurun_out/carveout.log; : > $out
for cv in unset 100 75; do
  if [ $cv = unset ]; then unset FIZI_CARVEOUT; else export FIZI_CARVEOUT=$cv; fi
  TL_CONFIG=3 TL_WARM=5 TL_NCALLS=20 timeout 300 python scripts/timeline.py > gpurun_out/tl_cv_$cv.log 2>&1
  for cfg in 3 4 2; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== carveout=$cv C$cfg" >> $out
    timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items() if v})" >> $out 2>&1
  done
  echo "== carveout=$cv C3 driver" >> $out
  for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out 2>&1
  done
done
