#!/bin/bash
# A/B: host entry chunk size (FIZI_HOST_CHUNK_MB) for the e2e leg
mkdir -p gpurun_out
out=gpurun_out/chunk_mb.log; : > $out
for mb in 32 8 16 64; do
  for cfg in 3 2 5; do
    echo "== chunk=${mb}MB C$cfg" >> $out
    FIZI_HOST_CHUNK_MB=$mb timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-spot-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['value']), d['e2e']['steps'])" >> $out 2>&1
  done
done
