#!/bin/bash
# C3 launch-parameter sweep of the fused kernel in the pipeline
mkdir -p gpurun_out
out=gpurun_out/c3_sweep2.log; : > $out
run() {
  echo "== $*" >> $out
  env "$@" timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1), 'seg_alone_joined', round(d['roofline']['stage_ms_per_step']['segment']*1e3,1))" >> $out 2>&1
}
run X=1
run FIZI_GROUP=16
run FIZI_GROUP=24
run FIZI_SEG_GRID=444
run FIZI_SEG_GRID=407
run FIZI_SEG_GRID=333
run X=1
