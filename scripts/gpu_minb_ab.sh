#!/bin/bash
# per-pixel word kernel occupancy A/B: default vs __launch_bounds__(256, 4 | 5) builds
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/minb_ab.log
cp paper_1907_04393_b200/libfizi.so /tmp/libfizi_def.so
for cfg in 4 3; do
  if [ $cfg = 4 ]; then P="python bench.py --config 4 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline"
  else P="python bench.py --config 3 --steps 300 --warmup 10 --no-e2e --no-cpu-baseline"; fi
  for v in def minb4 minb5 def minb4; do
    if [ $v = def ]; then cp /tmp/libfizi_def.so paper_1907_04393_b200/libfizi.so
    else cp paper_1907_04393_b200/libfizi_$v.so paper_1907_04393_b200/libfizi.so; fi
    echo "=== C$cfg $v" >> gpurun_out/minb_ab.log
    timeout 600 $P 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items()})" >> gpurun_out/minb_ab.log 2>&1
  done
done
cp /tmp/libfizi_def.so paper_1907_04393_b200/libfizi.so
