#!/bin/bash
# A/B: non-persistent fused kernel (one CTA per item) + stream priorities, so
# that the tail stages' CTAs are dispatched ahead of the fused kernel's
mkdir -p gpurun_out
out=gpurun_out/prio_ab.log; : > $out
run() {
  for cfg in 4 2 3; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== $* C$cfg" >> $out
    env "$@" timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'seg', round(d['roofline']['kernel_ms_per_step']*1e3,1))" >> $out 2>&1
  done
}
run X=1
run FIZI_SEG_PERSIST=0
run FIZI_SEG_PERSIST=0 FIZI_HEAD_PRIO=0
run FIZI_SEG_PERSIST=0 FIZI_SIDE_PRIO=1
run FIZI_HEAD_PRIO=0
