#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/ccl_threads.log; : > $out
for t in 512 256 1024; do
  for cfg in 3 4 5; do
    st=100; [ $cfg = 4 ] && st=40
    echo "== ccl threads=$t C$cfg" >> $out
    FIZI_CCL_THREADS=$t timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'ccl', round(d['roofline']['stage_ms_per_step']['ccl']*1e3,1))" >> $out 2>&1
  done
done
