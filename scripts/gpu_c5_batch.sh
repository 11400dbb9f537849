#!/bin/bash
# C5: frames per call (one frame from each of B streams)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/c5_batch.log
for b in 32 64 128 256; do
  echo "=== B=$b" >> gpurun_out/c5_batch.log
  timeout 600 python bench.py --config 5 --batch $b --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step']*1e3,1), round(r['frac'],3), round(r['step']['frac'],3), {k: round(v*1e3,1) for k,v in r['stage_ms_per_step'].items()})" >> gpurun_out/c5_batch.log 2>&1
done
