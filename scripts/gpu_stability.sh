#!/bin/bash
# run-to-run spread of the bench line: 6 x the driver's command, 3 x the default run (C3)
mkdir -p gpurun_out
out=gpurun_out/stability.log; : > $out
for i in 1 2 3 4 5 6; do
  timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('driver', round(d['value']), round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $out 2>&1
done
for i in 1 2 3; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', round(d['value']), round(d['ms_per_step']*1e3,1), d['steps'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['host_step_gaps']['max_us'])" >> $out 2>&1
done
