#!/bin/bash
# C3 / C5: per-pixel word kernel, ALU test (default) vs colour-table build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/slow_ab3.log
for cfg in 3 5; do
P="python bench.py --config $cfg --steps 300 --warmup 10 --no-e2e --no-cpu-baseline"
for r in 1 2; do
  echo "=== C$cfg alu" >> gpurun_out/slow_ab3.log
  timeout 600 $P 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['stage_ms_per_step'])" >> gpurun_out/slow_ab3.log 2>&1
  cp paper_1907_04393_b200/libfizi.so /tmp/libfizi_keep.so
  cp paper_1907_04393_b200/libfizi_table.so paper_1907_04393_b200/libfizi.so
  echo "=== C$cfg table" >> gpurun_out/slow_ab3.log
  timeout 600 $P 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['stage_ms_per_step'])" >> gpurun_out/slow_ab3.log 2>&1
  cp /tmp/libfizi_keep.so paper_1907_04393_b200/libfizi.so
done
done
