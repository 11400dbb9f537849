#!/bin/bash
# C4: the fused kernel's persistent grid vs the co-running per-pixel words stage
mkdir -p gpurun_out
out=gpurun_out/c4_sweep.log; : > $out
run() {
  echo "== $*" >> $out
  env "$@" timeout 300 python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1), 'stages', {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items() if v})" >> $out 2>&1
}
run X=1
run FIZI_SEG_GRID=296
run FIZI_SEG_GRID=222
run FIZI_SEG_GRID=148
run FIZI_SIDE_PRIO=1
run FIZI_SEG_GRID=296 FIZI_SIDE_PRIO=1

for g in 296 222; do
  echo "== C3 grid $g" >> $out
  FIZI_SEG_GRID=$g timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out
done
echo "== C3 default" >> $out
timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))" >> $out
